"""GPU calibration (K6) and DP allocation (K7/K8) vs the oracle."""
import numpy as np
import pytest
import torch

from tests import gpu_env as E

pytestmark = pytest.mark.gpu

from oracle import dp as ODP
from oracle import pca as OPCA
from oracle import quant as OQ
from kvtc_inputs import generate, sample_positions


@pytest.fixture(scope="module")
def K():
    from paper_2511_01815_b200 import kvtc
    kvtc.device_check()
    return kvtc


def _rand_P(rng, n, r, ties=False):
    scale = (1.0 + np.arange(r)) ** -0.8 * 3.0
    P = rng.standard_normal((n, r)) * scale + rng.normal(0, 0.3, (1, r))
    if ties:
        P = np.round(P * 4) / 4
    return P.astype(np.float32)


CASES = [
    # (n, r, B, sizes, type_mask)
    (512, 200, 1000, (1, 16, 64, 256, 1024), 0xF),
    (100, 64, 501, (1, 16, 64), 0xF),
    (37, 40, 300, (1, 2, 4), 0x7),
    (64, 33, 260, (1, 2, 4, 16), 0xB),
    (1000, 130, 2048, (1, 16, 64, 256, 1024), 0xF),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_dp_bitexact_vs_literal_loop(K, case):
    n, r, B, sizes, mask = CASES[case]
    rng = np.random.default_rng(case)
    P = _rand_P(rng, n, r, ties=case == 3)
    types = tuple(t for t in OQ.TYPES if t == 0 or (mask >> t) & 1)
    ref = ODP.dp_literal_c(P.astype(np.float64), B, sizes, types)
    Pd = torch.from_numpy(P).cuda()
    got = K.dp_best_table(Pd, B, sizes, mask).cpu().numpy()
    np.testing.assert_array_equal(got, ref.best[:, 0::2][:, : got.shape[1]])
    # the plan from the full entry point == the oracle's backtrack, bit for bit
    plan = K.allocate_bits_from_coeffs(Pd, p_original=B, target_cr=16.0, sizes=sizes,
                                       type_mask=mask)
    info = plan.info()
    oplan = ODP.backtrack(ref, B)
    assert info.budget == B
    assert info.groups == [tuple(g) for g in oplan.groups]
    assert info.expected_error == ref.best[r, B]


def test_dp_on_calibrated_coefficients(K):
    """Real DP input: the toy oracle basis' coefficients, headline CR 16."""
    spec, invf, kb, vb, Ck, Cv = E.setup("toy")
    for ob, C0 in ((kb, Ck), (vb, Cv)):
        P = OPCA.dp_coefficients(ob, C0).astype(np.float32)
        for cr in (8, 16, 32):
            oplan, res, B = ODP.allocate(P.astype(np.float64), cr, spec.p)
            plan = K.allocate_bits_from_coeffs(torch.from_numpy(P).cuda(), spec.p, cr)
            info = plan.info()
            assert info.groups == [tuple(g) for g in oplan.groups], (cr, info.groups, oplan.groups)
            assert info.expected_error == res.best[-1, B]


def test_multi_cr_plans_equal_oracle_plans(K):
    """One DP table at the largest budget, one backtrack per CR (kvtc_allocate_bits_
    from_coeffs_multi) == the oracle's DP run separately at every CR."""
    spec, invf, kb, vb, Ck, Cv = E.setup("toy")
    P = OPCA.dp_coefficients(kb, Ck).astype(np.float32)
    crs = [32.0, 4.0, 16.0, 8.0, 12.5]
    plans = K.allocate_bits_from_coeffs_multi(torch.from_numpy(P).cuda(), spec.p, crs)
    for cr, plan in zip(crs, plans):
        oplan, res, B = ODP.allocate(P.astype(np.float64), cr, spec.p)
        info = plan.info()
        assert info.budget == B
        assert info.groups == [tuple(g) for g in oplan.groups], cr
        assert info.expected_error == res.best[-1, B]


@pytest.mark.parametrize("name", ["toy", "mid"])
def test_calibrate_vs_oracle(K, name):
    spec, invf, kb, vb, Ck, Cv = E.setup(name)
    tcal = 2048 if name == "toy" else 3200
    ncal = 2000 if name == "toy" else 3000
    cal = [generate(spec, st, tcal, pos0=0, conversation=100).cuda() for st in (0, 1)]
    samples = sample_positions([tcal], ncal, sinks=spec.sinks, seed=1)
    for which, ob in ((0, kb), (1, vb)):
        B = K.calibrate([K.KVView(cal[which])], samples, which, 10000, inv_freq=invf.astype(np.float32))
        mu, V, sg = B.get()
        assert V.shape == ob.V.shape
        np.testing.assert_allclose(mu, ob.mu, rtol=1e-5, atol=1e-6 * np.abs(ob.mu).max())
        k = min(spec.latent, 64)
        np.testing.assert_allclose(sg[:k], ob.sigma[:k], rtol=2e-4)
        # leading principal directions agree (up to the canonical sign, which both apply)
        cos = np.abs(np.sum(V[:, :k].astype(np.float64) * ob.V[:, :k], axis=0))
        gaps = np.abs(np.diff(ob.sigma[: k + 1] ** 2))
        well = gaps[:k] > 1e-3 * ob.sigma[0] ** 2
        assert np.all(cos[well] > 0.999), cos[well].min()
        np.testing.assert_array_less(-1e-6, np.sum(V[:, :k] * ob.V[:, :k], axis=0)[well])


def test_randomized_svd_path(K, monkeypatch):
    """The large-p finalize path (randomized SVD, P:L235, 8 power iterations,
    P:L974) forced on the mid shape: leading directions match the oracle."""
    monkeypatch.setenv("KVTC_CALIB_RSVD", "1")
    spec, invf, kb, vb, Ck, Cv = E.setup("mid")
    cal = generate(spec, 1, 3200, pos0=0, conversation=100).cuda()
    samples = sample_positions([3200], 3000, sinks=spec.sinks, seed=1)
    B = K.calibrate([K.KVView(cal)], samples, 1, 256)
    mu, V, sg = B.get()
    assert V.shape == (spec.p, 256)
    k = 64
    np.testing.assert_allclose(sg[:k], vb.sigma[:k], rtol=1e-3)
    cos = np.abs(np.sum(V[:, :k].astype(np.float64) * vb.V[:, :k], axis=0))
    gaps = np.abs(np.diff(vb.sigma[: k + 1] ** 2))
    well = gaps[:k] > 1e-2 * vb.sigma[0] ** 2
    assert np.all(cos[well] > 0.99), cos[well].min()


def _golden_dp():
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "dp_production.json")) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("case", ["decay_b32768", "tail_1024", "tail_256"])
def test_dp_bitexact_at_production_shape(K, case):
    """the 256- and 1024-block E-table paths and the scan over 16,385
    even budgets (B = 32768, the Llama-8B budget at CR 16) against the literal
    loop of P:L1541-1603.  Expected values: tests/golden/dp_production.json,
    written by scripts/make_dp_golden.py from oracle/ only (oracle DP on the same
    seeded inputs); the GPU's even-budget best_error table must hash identically
    and the backtracked plan and best_error[r][B] must be equal."""
    import hashlib
    from kvtc_inputs import dp_coefficients
    g = _golden_dp()[case]
    prm = g["params"]
    B = prm["budget"]
    P = dp_coefficients(**prm)
    Pd = torch.from_numpy(P).cuda()
    got = K.dp_best_table(Pd, B).cpu().numpy()
    assert list(got.shape) == g["best_even_shape"]
    if hashlib.sha256(np.ascontiguousarray(got).astype("<f8").tobytes()).hexdigest() != g["best_even_sha256"]:
        r = P.shape[1]
        step = max(1, got.shape[1] // 16)
        for i, row in g["rows_hex"].items():
            np.testing.assert_array_equal(got[int(i), ::step], [float.fromhex(v) for v in row], err_msg=f"row {i}")
        raise AssertionError("best_error table differs from the oracle's (rows sampled above agree)")
    plan = K.allocate_bits_from_coeffs(Pd, p_original=B, target_cr=16.0)
    info = plan.info()
    assert info.budget == B
    assert info.groups == [tuple(x) for x in g["groups"]]
    assert info.expected_error == float.fromhex(g["expected_error_hex"])
    assert set(z for (_, z, _) in info.groups) >= set(g["sizes_in_plan"]) - {1}
