"""Pins for oracle/pca.py and oracle/codec.py."""
import zlib

import numpy as np
import pytest
import torch

from oracle import codec as C
from oracle import dp as DP
from oracle import pca as PCA
from oracle import quant as Q
from oracle import entropy
from kvtc_inputs import make_spec, generate, sample_positions


def test_kv_cache_bytes_table1():
    MiB = 1 << 20
    assert C.kv_cache_bytes(32, 8, 128, 1024) == 128 * MiB      # Llama 3.1 8B
    assert C.kv_cache_bytes(80, 8, 128, 1024) == 320 * MiB      # Llama 3.3 70B
    assert C.kv_cache_bytes(40, 8, 128, 1024) == 160 * MiB      # Mistral NeMo 12B
    assert C.kv_cache_bytes(28, 2, 128, 1024) == 28 * MiB       # Qwen 2.5 R1 1.5B
    assert C.kv_cache_bytes(28, 4, 128, 1024) == 56 * MiB       # Qwen 2.5 R1 7B


def test_pca_against_svd_and_orthonormality():
    rng = np.random.default_rng(0)
    C0 = rng.standard_normal((300, 40)) @ rng.standard_normal((40, 40)) + 3.0
    b = PCA.fit(C0, 40)
    np.testing.assert_allclose(b.V.T @ b.V, np.eye(40), atol=1e-6)
    s = np.linalg.svd(C0 - C0.mean(axis=0), compute_uv=False)
    np.testing.assert_allclose(b.sigma, s, rtol=1e-9)
    np.testing.assert_allclose(b.mu, C0.mean(axis=0), rtol=1e-6)
    # canonical sign: the largest-|entry| of each column is positive
    idx = np.argmax(np.abs(b.V), axis=0)
    assert np.all(b.V[idx, np.arange(40)] > 0)


def test_planted_rank_and_full_rank_identity():
    rng = np.random.default_rng(1)
    F = rng.standard_normal((500, 5)) @ rng.standard_normal((5, 30))
    b = PCA.fit(F, 30)
    # covariance route: sigma of a zero direction is O(sqrt(eps))*sigma_0
    assert np.sum(b.sigma > 1e-5 * b.sigma[0]) == 5
    # full-rank fp64 basis: project -> reconstruct is the identity
    w, V = np.linalg.eigh(np.cov(F.T))
    X = rng.standard_normal((7, 30))
    mu = F.mean(axis=0)
    D = (X - mu) @ V
    np.testing.assert_allclose(D @ V.T + mu, X, atol=1e-10)
    # truncation error == sum of discarded squared coefficients
    k = 12
    err = np.sum((D[:, :k] @ V[:, :k].T + mu - X) ** 2)
    assert err == pytest.approx(np.sum(D[:, k:] ** 2), rel=1e-9)


def test_orthonormal_invariance():
    """P:L246-250 / SPEC acceptance 2: ||D V^T - D_q V^T||_F = ||D - D_q||_F."""
    rng = np.random.default_rng(2)
    for _ in range(100):
        p, r = int(rng.integers(5, 60)), None
        r = int(rng.integers(1, p + 1))
        V, _ = np.linalg.qr(rng.standard_normal((p, r)))
        D = rng.standard_normal((9, r))
        Dq = D + rng.standard_normal((9, r)) * 0.1
        assert np.linalg.norm(D @ V.T - Dq @ V.T) == pytest.approx(np.linalg.norm(D - Dq), rel=1e-9)


def test_zlib_roundtrip():
    rng = np.random.default_rng(3)
    for n in (0, 1, 1000, 65536, 200000):
        buf = rng.integers(0, 4, n, dtype=np.uint8).tobytes()
        ch = entropy.deflate_chunks(buf)
        assert entropy.inflate_chunks(ch) == buf
        assert all(len(zlib.decompress(c, wbits=-15)) <= entropy.CHUNK_BYTES for c in ch)


def _toy_setup(cr_list=(16,)):
    spec = make_spec("toy")
    invf = spec.inv_freq().double().numpy()
    cal = [(generate(spec, st, 2048, pos0=0, conversation=100).double().numpy(), 0) for st in (0, 1)]
    samples = sample_positions([2048], 2000, sinks=4, seed=0)
    Ck = PCA.gather([cal[0]], samples, True, invf)
    Cv = PCA.gather([cal[1]], samples, False)
    kb, vb = PCA.fit(Ck, 10000), PCA.fit(Cv, 10000)
    return spec, invf, kb, vb, Ck, Cv


@pytest.fixture(scope="module")
def toy():
    return _toy_setup()


def test_end_to_end_toy(toy):
    spec, invf, kb, vb, Ck, Cv = toy
    Pk, Pv = PCA.dp_coefficients(kb, Ck), PCA.dp_coefficients(vb, Cv)
    t, pos0 = 512, 0
    K = generate(spec, 0, t, pos0=pos0, conversation=0).double().numpy()
    V = generate(spec, 1, t, pos0=pos0, conversation=0).double().numpy()
    errs = []
    for cr in (64, 32, 16, 8, 4):   # toy p=128: CR 64 -> B=32 < 34, all-None plan
        kp, _, Bk = DP.allocate(Pk, cr, spec.p)
        vp, _, Bv = DP.allocate(Pv, cr, spec.p)
        assert kp.bits_per_token <= Bk and vp.bits_per_token <= Bv
        c = C.compress(K, V, pos0, kb, kp, vb, vp, invf)
        assert c.stats["cr_pre_deflate"] >= cr * (1 - 1e-9)
        K2, V2 = C.decompress(c, kb, kp, vb, vp, invf)
        # sinks and window byte-identical
        np.testing.assert_array_equal(K2[:, :4], K[:, :4])
        np.testing.assert_array_equal(K2[:, -128:], K[:, -128:])
        np.testing.assert_array_equal(V2[:, :4], V[:, :4])
        np.testing.assert_array_equal(V2[:, -128:], V[:, -128:])
        mid = slice(4, t - 128)
        e = (np.linalg.norm(K2[:, mid] - K[:, mid]) / np.linalg.norm(K[:, mid]),
             np.linalg.norm(V2[:, mid] - V[:, mid]) / np.linalg.norm(V[:, mid]))
        errs.append(e)
    ek = [e[0] for e in errs]
    ev = [e[1] for e in errs]
    # error non-increasing as the target CR decreases (SPEC acceptance 7)
    assert all(a >= b * (1 - 1e-6) for a, b in zip(ek, ek[1:]))
    assert all(a >= b * (1 - 1e-6) for a, b in zip(ev, ev[1:]))
    assert ek[-1] < 0.1 and ev[-1] < 0.1


def test_nothing_to_compress(toy):
    spec, invf, kb, vb, Ck, Cv = toy
    K = generate(spec, 0, 132, conversation=3).double().numpy()
    V = generate(spec, 1, 132, conversation=3).double().numpy()
    plan = DP.Plan(r=kb.r, blocks=[])
    c = C.compress(K, V, 0, kb, plan, vb, plan, invf)
    assert c.stats.get("nothing_to_compress")
    K2, V2 = C.decompress(c, kb, plan, vb, plan, invf)
    np.testing.assert_array_equal(K2, K)
    np.testing.assert_array_equal(V2, V)


def _exact_basis():
    """An orthonormal, NON-symmetric 4x4 basis whose entries (+-1/2) are exact in
    bf16 and fp16, so V_c = V_d = V and every step below is exact in fp64: the
    Hadamard matrix / 2 with its columns permuted (2, 0, 3, 1)."""
    H = 0.5 * np.array([[1, 1, 1, 1], [1, -1, 1, -1], [1, 1, -1, -1], [1, -1, -1, 1]], dtype=np.float64)
    V = H[:, [2, 0, 3, 1]]
    mu = np.array([1.0, 2.0, 3.0, 4.0])
    return PCA.Basis(mu=mu, V=V, sigma=np.ones(4), n=0), V, mu


def test_project_worked_example():
    """D = (X - mu) V.  Worked by hand: X - mu = [2, 0, 0, 0] gives
    2 * (row 0 of V) = [1, 1, 1, 1]; X - mu = [0, 2, 0, 0] gives 2 * row 1 =
    [1, 1, -1, -1]; X = mu gives 0 (a dropped mu V_c term fails this);
    X - mu = [0, 0, 0, 4] gives 4 * row 3 = [-2, 2, 2, -2] (a transposed V
    fails, V is not symmetric)."""
    b, V, mu = _exact_basis()
    X = mu[None, :] + np.array([[2.0, 0, 0, 0], [0, 2.0, 0, 0], [0, 0, 0, 0], [0, 0, 0, 4.0]])
    D = PCA.project(b, X)
    np.testing.assert_array_equal(D, [[1, 1, 1, 1], [1, 1, -1, -1], [0, 0, 0, 0], [-2, 2, 2, -2]])
    # a column subset projects onto those PCs only
    np.testing.assert_array_equal(PCA.project(b, X, cols=[3, 1]), D[:, [3, 1]])


def test_reconstruct_inverts_projection_and_truncation_error():
    """X = D V^T + mu with all p PCs (exact here: V^T V = I);
    keeping a subset of PCs leaves ||X - X^||^2 = the sum of the discarded
    squared coefficients (orthonormal invariance)."""
    b, V, mu = _exact_basis()
    rng = np.random.default_rng(3)
    X = mu[None, :] + rng.integers(-8, 9, (5, 4)).astype(np.float64)
    D = PCA.project(b, X)
    np.testing.assert_array_equal(PCA.reconstruct(b, D), X)
    keep = [0, 2]
    Xh = PCA.reconstruct(b, D[:, keep], cols=keep)
    np.testing.assert_array_equal(np.sum((X - Xh) ** 2, axis=1), np.sum(D[:, [1, 3]] ** 2, axis=1))


def test_fit_svd_equals_fit():
    """fit_svd (SVD of C - mu, P:L226-229 literally) and fit (eigh of the
    covariance) give the same sigma and, where the spectrum has gaps, the same
    directions with the same canonical sign."""
    rng = np.random.default_rng(5)
    n, p = 300, 40
    A = rng.standard_normal((n, p)) * (1.0 + np.arange(p)) ** -1.0 * 4 + rng.normal(0, 1, p)
    a, b = PCA.fit(A, 30), PCA.fit_svd(A, 30)
    np.testing.assert_allclose(b.sigma, a.sigma, rtol=1e-10)
    np.testing.assert_array_equal(a.mu, b.mu)
    np.testing.assert_allclose(b.V, a.V, atol=2e-6)       # both fp32 masters


def test_project_partial_block_identity():
    """Q23: the shards' partial projections sum to the projection of the joint
    features, D = sum_g X_g V_g - mu V (the block-matrix identity), checked against
    the joint project() for an uneven split into three layer shards."""
    rng = np.random.default_rng(23)
    n, p, r = 50, 96, 10
    X = rng.standard_normal((n, p))
    C = rng.standard_normal((200, p)) @ rng.standard_normal((p, p)) * 0.1
    b = PCA.fit(C, r)
    cols = np.arange(0, r, 2)
    splits = [(0, 32), (32, 40), (40, 96)]
    parts = [PCA.project_partial(b, X[:, f0:f1], f0, f1, k == 0, cols) for k, (f0, f1) in enumerate(splits)]
    np.testing.assert_allclose(sum(parts), PCA.project(b, X, cols), rtol=1e-12, atol=1e-12)
    # the mean enters once: without any bias the sum is X V, not (X - mu) V
    no_bias = sum(PCA.project_partial(b, X[:, f0:f1], f0, f1, False, cols) for (f0, f1) in splits)
    np.testing.assert_allclose(no_bias - PCA.project(b, X, cols), np.tile(b.mu @ b.Vc[:, cols], (n, 1)),
                               rtol=1e-12, atol=1e-12)
