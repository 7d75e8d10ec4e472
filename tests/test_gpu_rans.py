"""rANS back-end (reading Q24): the GPU section is bit-identical
to the oracle's encoding (frequency tables, chunk kinds and streams), the GPU
decoder restores the bytes of its own and of the oracle's sections, and a
damaged stream is reported as KVTC_E_CORRUPT."""
import numpy as np
import pytest
import torch

from oracle import rans as OR
from tests import gpu_env as E
from tests.kvtc_format import build_rans_section, parse_rans_section

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    from paper_2511_01815_b200 import kvtc
    kvtc.device_check()
    return kvtc


def _periodic(n, period, seed):
    rng = np.random.default_rng(seed)
    idx = np.arange(n)
    p = period or n
    skew = (idx % p) * 7 // max(1, p)
    return ((rng.geometric(0.2 + 0.1 * (skew % 3), n) + 17 * skew) % 256).astype(np.uint8)


def _check(K, data: np.ndarray, period: int, chunk: int):
    t = torch.from_numpy(data).cuda()
    sec = K.rans_encode(t, period, chunk)
    buf = sec.cpu().numpy().tobytes()
    info = parse_rans_section(buf)
    freqs, sl, chunks = OR.encode(data.tobytes(), chunk, period)
    np.testing.assert_array_equal(info["freqs"], freqs)
    assert info["span_log2"] == sl and info["nchunks"] == len(chunks)
    for i, ((kg, sg), (ko, so)) in enumerate(zip(info["streams"], chunks)):
        assert kg == ko and sg == so, i                          # bit-exact streams
    assert K.rans_decode(sec, len(data)).cpu().numpy().tobytes() == data.tobytes()
    osec = torch.frombuffer(bytearray(build_rans_section(freqs, sl, chunks, len(data), chunk, period)),
                            dtype=torch.uint8).cuda()
    assert K.rans_decode(osec, len(data)).cpu().numpy().tobytes() == data.tobytes()
    return info


@pytest.mark.parametrize("n,period,chunk", [(200000, 0, 65536), (150000, 20000, 16384), (4097, 0, 65536),
                                            (70000, 3000, 32768), (33, 0, 65536)])
def test_rans_synthetic_vs_oracle(K, n, period, chunk):
    _check(K, _periodic(n, period, n), period, chunk)


def test_rans_incompressible_and_constant(K):
    rng = np.random.default_rng(1)
    n = 100000
    info = _check(K, rng.integers(0, 256, n).astype(np.uint8), 0, 65536)
    # random bytes: every chunk is stored or coded smaller than stored; the section
    # exceeds the raw bytes by its tables and tables of contents only
    assert all(len(st) <= 65536 for _, st in info["streams"])
    assert info["total"] <= n + 64 + info["nclasses"] * 512 + 16 * info["nchunks"] + 16 * info["nchunks"] + 32
    info = _check(K, np.full(70000, 7, np.uint8), 0, 65536)    # one symbol: f = M, no words at all
    assert all(k == 0 and len(st) == 128 for k, st in info["streams"])


def test_rans_on_codec_payload(K):
    """The mid config's packed payload (tile period = the plan's tile bytes)."""
    spec, invf, kb, vb, Ck, Cv = E.setup("mid")
    groups = E.mid_plan_groups()
    shape = (spec.layers, spec.kv_heads, spec.head_dim)
    B = K.Basis.create(shape, 1, vb.mu, vb.V, vb.sigma)
    Pl = K.Plan.create(vb.r, groups)
    _, Vc = E.caches("mid", 3000, 0)
    X = K.gather(K.KVView(Vc.cuda()), 4, 3000 - 132, False)
    payload = K.project_quantize(B, Pl, X).cpu().numpy()
    tile = Pl.payload_bytes(128)
    info = _check(K, payload, tile, 65536)
    assert info["period"] == tile


def test_rans_corrupt_stream_reported(K):
    data = _periodic(100000, 0, 5)
    sec = K.rans_encode(torch.from_numpy(data).cuda(), 0, 65536)
    info = parse_rans_section(sec.cpu().numpy().tobytes())
    k0, s0 = info["streams"][0]
    assert k0 == 0
    off = info["data_off"] + int(info["table"][0]["off"]) + 200        # a word of chunk 0
    bad = sec.clone()
    bad[off] ^= 0x5A
    from paper_2511_01815_b200 import _lib as L
    with pytest.raises(L.KvtcError) as e:
        K.rans_decode(bad, len(data))
    assert e.value.status == -3                                     # KVTC_E_CORRUPT
