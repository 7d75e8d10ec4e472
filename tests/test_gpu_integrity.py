"""The boundary's error contract (include/kvtc.h, SURVEY §8(b) conventions):
KVTC_E_CORRUPT for damaged containers, KVTC_E_NUMERIC for 16-bit factor
overflow (reading Q4), KVTC_E_MISMATCH for a basis / plan the container was not
written with.  "This step is lossless": after any byte flip, the
decompressor either restores exactly what the intact container restores, or
fails loudly; it never writes garbage with KVTC_OK and never faults."""
import numpy as np
import pytest
import torch

from tests import gpu_env as E
from tests.kvtc_format import parse_container, parse_section

pytestmark = pytest.mark.gpu

from oracle import codec as OC
from oracle import dp as ODP

CORRUPT, NUMERIC, MISMATCH = -3, -2, -4


@pytest.fixture(scope="module")
def K():
    from paper_2511_01815_b200 import kvtc
    kvtc.device_check()
    return kvtc


@pytest.fixture(scope="module")
def mid(K):
    """The mid shape (p = 2048, 4 DEFLATE chunks per stream) and one container."""
    spec, invf, kb, vb, Ck, Cv = E.setup("mid")
    shape = (spec.layers, spec.kv_heads, spec.head_dim)
    g = E.mid_plan_groups()
    KB = K.Basis.create(shape, 0, kb.mu, kb.V, kb.sigma, inv_freq=invf, pairing=0)
    VB = K.Basis.create(shape, 1, vb.mu, vb.V, vb.sigma)
    KP = K.Plan.create(kb.r, g)
    VP = K.Plan.create(vb.r, g)
    t, pos0 = 1000, 300
    Kc, Vc = E.caches("mid", t, pos0, conversation=11)
    kd, vd = Kc.cuda(), Vc.cuda()
    cont, st = K.compress(KB, KP, VB, VP, K.KVView(kd, pos0=pos0), K.KVView(vd, pos0=pos0))
    ref_k, ref_v = torch.zeros_like(kd), torch.zeros_like(vd)
    K.decompress(KB, KP, VB, VP, cont, K.KVView(ref_k, pos0=pos0), K.KVView(ref_v, pos0=pos0))
    torch.cuda.synchronize()
    return dict(spec=spec, invf=invf, kb=kb, vb=vb, KB=KB, VB=VB, KP=KP, VP=VP, t=t, pos0=pos0, kd=kd, vd=vd,
                cont=cont, ref_k=ref_k, ref_v=ref_v)


def _outs(M):
    return torch.zeros_like(M["kd"]), torch.zeros_like(M["vd"])


def _decompress_status(K, M, cont, in_len=None):
    """(status, k_out, v_out) of the synchronous decompress of `cont`."""
    ko, vo = _outs(M)
    try:
        if in_len is not None:
            cont = cont[:in_len]
        K.decompress(M["KB"], M["KP"], M["VB"], M["VP"], cont, K.KVView(ko, pos0=M["pos0"]),
                     K.KVView(vo, pos0=M["pos0"]))
        torch.cuda.synchronize()
        return 0, ko, vo
    except K.KvtcError as e:
        return e.status, ko, vo


def test_async_decompress_equals_sync_and_reports_ok(K, mid):
    M = mid
    hdr = M["cont"][:256].cpu().numpy().tobytes()
    status = torch.full((1,), 12345, dtype=torch.int32, device="cuda")
    ko, vo = _outs(M)
    K.decompress_async(M["KB"], M["KP"], M["VB"], M["VP"], M["cont"], hdr, K.KVView(ko, pos0=M["pos0"]),
                       K.KVView(vo, pos0=M["pos0"]), status)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    assert torch.equal(ko, M["ref_k"]) and torch.equal(vo, M["ref_v"])
    info = K.container_info(M["cont"])
    assert info.flags == 0 and info.raw_hash != 0


def _regions(buf):
    h = parse_container(buf)
    regions = {"header": (0, 256), "raw": (256, 256 + h["raw_bytes"])}
    for nm, key in (("k", "sec_k"), ("v", "sec_v")):
        sec = parse_section(buf[h[key]:])
        off = h[key]
        nch = sec["nchunks"]
        regions[f"{nm}.sec_header"] = (off, off + 64)
        regions[f"{nm}.chunk_table"] = (off + 64, off + 64 + 16 * nch)
        regions[f"{nm}.index"] = (off + 64 + 16 * nch, off + sec["data_off"])
        regions[f"{nm}.streams"] = (off + sec["data_off"], off + sec["total"])
    return regions


def test_byte_flip_fuzz(K, mid):
    """Random single-byte flips in every region of the container: the result is
    KVTC_E_CORRUPT or an exact restore (flips in alignment padding change
    nothing).  Never KVTC_OK with different output, never a device fault."""
    M = mid
    buf = M["cont"].cpu().numpy().tobytes()
    regions = _regions(buf)
    rng = np.random.default_rng(2024)
    outcomes = {}
    for name, (a, b) in regions.items():
        n_try = 6 if name in ("raw", "k.streams", "v.streams") else 4
        for _ in range(n_try):
            pos = int(rng.integers(a, b))
            bad = bytearray(buf)
            bad[pos] ^= int(rng.integers(1, 256))
            dev = torch.frombuffer(bad, dtype=torch.uint8).cuda()
            st, ko, vo = _decompress_status(K, M, dev)
            exact = st == 0 and torch.equal(ko, M["ref_k"]) and torch.equal(vo, M["ref_v"])
            assert st in (CORRUPT, MISMATCH) or exact, (name, pos, st)
            outcomes.setdefault(name, []).append("exact" if exact else {CORRUPT: "corrupt", MISMATCH: "mismatch"}[st])
    print("\n[fuzz]", outcomes)
    # every flip inside a checksummed byte range must be detected
    for name in ("header", "raw"):
        assert all(o != "exact" for o in outcomes[name]), (name, outcomes[name])
    # the device is still healthy: the intact container decompresses exactly
    st, ko, vo = _decompress_status(K, M, M["cont"])
    assert st == 0 and torch.equal(ko, M["ref_k"]) and torch.equal(vo, M["ref_v"])


def test_every_payload_flip_is_detected(K, mid):
    """Flips of stream bytes that the DEFLATE decoder would accept (same code
    length) are caught by the payload checksum: sweep the first data bytes of a
    stream, bit by bit."""
    M = mid
    buf = M["cont"].cpu().numpy().tobytes()
    h = parse_container(buf)
    sec = parse_section(buf[h["sec_v"]:])
    e = sec["table"][1]
    start = h["sec_v"] + sec["data_off"] + int(e["off"]) + 600          # past the block header
    for k in range(24):
        bad = bytearray(buf)
        bad[start + k // 8] ^= 1 << (k % 8)
        st, ko, vo = _decompress_status(K, M, torch.frombuffer(bad, dtype=torch.uint8).cuda())
        assert st == CORRUPT, (k, st)


def test_truncated_and_foreign_containers(K, mid):
    M = mid
    n = M["cont"].numel()
    for cut in (100, 256, n // 2, n - 1):
        st, _, _ = _decompress_status(K, M, M["cont"], in_len=cut)
        assert st in (CORRUPT, -1), (cut, st)          # E_INVALID for shorter than a header
    # a header from another container (different pos0 -> different raw / payloads)
    Kc, Vc = E.caches("mid", M["t"], 0, conversation=12)
    other, _ = K.compress(M["KB"], M["KP"], M["VB"], M["VP"], K.KVView(Kc.cuda()), K.KVView(Vc.cuda()))
    hdr = other[:256].cpu().numpy().tobytes()
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    ko, vo = _outs(M)
    try:
        K.decompress_async(M["KB"], M["KP"], M["VB"], M["VP"], M["cont"], hdr, K.KVView(ko, pos0=M["pos0"]),
                           K.KVView(vo, pos0=M["pos0"]), status)
        torch.cuda.synchronize()
        assert int(status.item()) == CORRUPT
    except K.KvtcError as e:
        assert e.status in (CORRUPT, MISMATCH)


def test_batch_reports_the_corrupt_item(K, mid):
    M = mid
    Kc, Vc = E.caches("mid", 600, 0, conversation=13)
    ks = [K.KVView(M["kd"], pos0=M["pos0"]), K.KVView(Kc.cuda())]
    vs = [K.KVView(M["vd"], pos0=M["pos0"]), K.KVView(Vc.cuda())]
    conts = K.compress_batch(M["KB"], M["KP"], M["VB"], M["VP"], ks, vs)
    assert torch.equal(conts[0], M["cont"])          # the batched container == the single call's
    buf = bytearray(conts[1].cpu().numpy().tobytes())
    h = parse_container(bytes(buf))
    buf[h["sec_k"] + 4000] ^= 0x10
    bad = torch.frombuffer(buf, dtype=torch.uint8).cuda()
    outs = [(torch.zeros_like(M["kd"]), torch.zeros_like(M["vd"])), (torch.zeros_like(Kc.cuda()), torch.zeros_like(Vc.cuda()))]
    with pytest.raises(K.KvtcError) as ei:
        K.decompress_batch(M["KB"], M["KP"], M["VB"], M["VP"], [conts[0], bad],
                           [K.KVView(outs[0][0], pos0=M["pos0"]), K.KVView(outs[1][0])],
                           [K.KVView(outs[0][1], pos0=M["pos0"]), K.KVView(outs[1][1])])
    assert ei.value.status == CORRUPT and "item 1" in str(ei.value)


def test_numeric_overflow_matches_oracle(K):
    """Q4: a coefficient range beyond binary16 makes the oracle raise
    (oracle/codec.py) and the GPU flag the container: compress returns
    KVTC_E_NUMERIC and so does decompress.  A large but representable range
    passes on both sides."""
    spec, invf, kb, vb, Ck, Cv = E.setup("toy")
    shape = (spec.layers, spec.kv_heads, spec.head_dim)
    kp, vp = E.toy_plans(16)
    KB = K.Basis.create(shape, 0, kb.mu, kb.V, kb.sigma, inv_freq=invf, pairing=0)
    VB = K.Basis.create(shape, 1, vb.mu, vb.V, vb.sigma)
    KP, VP = K.Plan.create(kb.r, kp.groups), K.Plan.create(vb.r, vp.groups)
    for scale, expect in ((3.0e2, 0), (3.0e5, NUMERIC)):
        Kc, Vc = E.caches("toy", 400, 0, conversation=21)
        Vc = Vc.clone()
        Vc[:, 200] = (Vc[:, 200].float() * scale).to(torch.bfloat16)      # one token's values blown up
        try:
            OC.compress(Kc.double().numpy(), Vc.double().numpy(), 0, kb, ODP.Plan(r=kb.r, blocks=list(kp.groups)),
                        vb, ODP.Plan(r=vb.r, blocks=list(vp.groups)), invf)
            oracle = 0
        except FloatingPointError:
            oracle = NUMERIC
        assert oracle == expect, (scale, oracle)
        try:
            cont, _ = K.compress(KB, KP, VB, VP, K.KVView(Kc.cuda()), K.KVView(Vc.cuda()))
            gpu = 0
        except K.KvtcError as e:
            gpu = e.status
        assert gpu == expect, (scale, gpu)
        if expect:
            # the container is written and flagged: decompress refuses it
            cont, _ = K.compress(KB, KP, VB, VP, K.KVView(Kc.cuda()), K.KVView(Vc.cuda()), sync_len=False)
            torch.cuda.synchronize()
            with pytest.raises(K.KvtcError) as ei:
                K.decompress(KB, KP, VB, VP, cont, K.KVView(torch.zeros_like(Kc.cuda())),
                             K.KVView(torch.zeros_like(Vc.cuda())))
            assert ei.value.status == NUMERIC


def test_rope_is_part_of_the_basis_fingerprint(K):
    """A key basis that differs only in its RoPE frequencies is a different
    transform: decompressing with it is KVTC_E_MISMATCH, not silent re-rotation
    with the wrong angles."""
    spec, invf, kb, vb, Ck, Cv = E.setup("toy")
    shape = (spec.layers, spec.kv_heads, spec.head_dim)
    kp, vp = E.toy_plans(16)
    KB = K.Basis.create(shape, 0, kb.mu, kb.V, kb.sigma, inv_freq=invf, pairing=0)
    KB2 = K.Basis.create(shape, 0, kb.mu, kb.V, kb.sigma, inv_freq=invf * 0.5, pairing=0)
    KB3 = K.Basis.create(shape, 0, kb.mu, kb.V, kb.sigma, inv_freq=invf, pairing=1)
    VB = K.Basis.create(shape, 1, vb.mu, vb.V, vb.sigma)
    KP, VP = K.Plan.create(kb.r, kp.groups), K.Plan.create(vb.r, vp.groups)
    Kc, Vc = E.caches("toy", 400, 0, conversation=22)
    cont, _ = K.compress(KB, KP, VB, VP, K.KVView(Kc.cuda()), K.KVView(Vc.cuda()))
    for other in (KB2, KB3):
        with pytest.raises(K.KvtcError) as ei:
            K.decompress(other, KP, VB, VP, cont, K.KVView(torch.zeros_like(Kc.cuda())),
                         K.KVView(torch.zeros_like(Vc.cuda())))
        assert ei.value.status == MISMATCH


def test_batch_async_per_item_status(K, mid):
    """kvtc_decompress_batch_async: no synchronisation, one verdict per item on
    the stream — the damaged item is flagged, the intact one restores exactly."""
    M = mid
    buf = bytearray(M["cont"].cpu().numpy().tobytes())
    h = parse_container(bytes(buf))
    buf[h["sec_v"] + 9000] ^= 0x01
    bad = torch.frombuffer(buf, dtype=torch.uint8).cuda()
    hdr = M["cont"][:256].cpu().numpy().tobytes()
    outs = [(torch.zeros_like(M["kd"]), torch.zeros_like(M["vd"])) for _ in range(2)]
    status = torch.full((2,), 77, dtype=torch.int32, device="cuda")
    K.decompress_batch_async(M["KB"], M["KP"], M["VB"], M["VP"], [M["cont"], bad], [hdr, hdr],
                             [K.KVView(o[0], pos0=M["pos0"]) for o in outs],
                             [K.KVView(o[1], pos0=M["pos0"]) for o in outs], status)
    torch.cuda.synchronize()
    assert status.tolist() == [0, CORRUPT]
    assert torch.equal(outs[0][0], M["ref_k"]) and torch.equal(outs[0][1], M["ref_v"])
