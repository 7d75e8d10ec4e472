"""The tests' own byte-format readers (tests/kvtc_format.py), pinned against
stock zlib on CPU before they are used to check GPU sections."""
import zlib

import numpy as np

from tests.kvtc_format import segment_bit_lengths, dynamic_header_bits


def test_segment_decoder_matches_zlib_huffman_only():
    rng = np.random.default_rng(0)
    for p, n, seg in ((0.1, 5000, 80), (0.02, 3000, 47), (0.5, 640, 10)):
        data = (rng.geometric(p, n) % 256).astype(np.uint8).tobytes()
        c = zlib.compressobj(6, zlib.DEFLATED, -15, 9, zlib.Z_HUFFMAN_ONLY)
        st = c.compress(data) + c.flush()
        lens, dec, end = segment_bit_lengths(st, len(data), seg, 64)
        assert dec == data                       # the literal decode agrees with zlib's encoder
        assert (end + 7) // 8 == len(st)         # final block ends in the last byte
        assert sum(lens) == end - dynamic_header_bits(st)
        assert all(x > 0 for x in lens[:-(-len(data) // seg)])
