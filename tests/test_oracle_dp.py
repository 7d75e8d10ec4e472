"""Pins for oracle/dp.py: brute force, base cases, invariants, C == Python."""
import numpy as np
import pytest

from oracle import dp as DP
from oracle import quant as Q


def _rand_P(rng, n, r):
    scale = (1.0 + np.arange(r)) ** -1.0 * rng.uniform(0.5, 5.0)
    return (rng.standard_normal((n, r)) * scale).astype(np.float32).astype(np.float64)


def test_dp_equals_brute_force():
    """SPEC acceptance 1 (the induction claim of P:L1604-1610 made executable):
    200 instances, r <= 8, batch <= 16, budget <= 128, sizes {1,2,4},
    types {None, int2, int4}; plus 40 instances that include fp8."""
    rng = np.random.default_rng(0)
    sizes = (1, 2, 4)
    for it in range(240):
        r = int(rng.integers(1, 9))
        n = int(rng.integers(1, 17))
        B = int(rng.integers(0, 129))
        types = (Q.T_NONE, Q.T_INT2, Q.T_INT4) if it < 200 else Q.TYPES
        P = _rand_P(rng, n, r)
        if it % 7 == 0:
            P[:, 0] = 3.0                                   # a constant column
        res = DP.dp_literal(P, B, sizes, types)
        bf, _ = DP.brute_force(P, B, sizes, types)
        assert res.best[r, B] == bf, (it, res.best[r, B], bf)
        plan = DP.backtrack(res, B)
        assert plan.bits_per_token <= B
        # folding the backtracked blocks reproduces the table value exactly
        Z, Qt = DP.ez_tables(P, sizes, types)
        v = res.init
        for (s0, z, t) in plan.blocks:
            si = sizes.index(z)
            v = (-Z[s0 + z, si] + Qt[s0 + z, si, types.index(t)]) + v
        assert v == res.best[r, B]


def test_base_cases_and_monotonicity():
    rng = np.random.default_rng(1)
    P = _rand_P(rng, 64, 40)
    res = DP.dp_literal(P, 400, (1, 16), Q.TYPES)
    init = DP.canonical_sq_sum(P)
    assert res.init == init
    assert np.all(res.best[0, :] == init) and np.all(res.best[:, 0] == init)
    assert np.all(np.diff(res.best, axis=1) <= 0)                              # non-increasing in b
    plan0 = DP.backtrack(res, 0)
    assert plan0.groups == []                                                  # zero budget: all None


def test_plan_error_matches_table_and_cost():
    rng = np.random.default_rng(2)
    P = _rand_P(rng, 128, 90)
    for B in (34, 100, 300, 700, 2000):
        res = DP.dp_literal(P, B, (1, 16, 64), Q.TYPES)
        plan = DP.backtrack(res, B)
        assert plan.bits_per_token <= B
        assert DP.plan_error(P, plan) == pytest.approx(res.best[-1, B], rel=1e-9, abs=1e-12)


def test_c_loop_equals_python_loop():
    rng = np.random.default_rng(3)
    for (n, r, B, sizes) in ((32, 70, 900, Q.SIZES), (16, 33, 501, (1, 16)), (8, 20, 0, (1,))):
        P = _rand_P(rng, n, r)
        ez = DP.ez_tables(P, sizes, Q.TYPES)
        a = DP.dp_literal(P, B, sizes, Q.TYPES, ez=ez)
        b = DP.dp_literal_c(P, B, sizes, Q.TYPES, ez=ez)
        np.testing.assert_array_equal(a.best, b.best)
        np.testing.assert_array_equal(a.btype, b.btype)
        np.testing.assert_array_equal(a.bsize, b.bsize)
        np.testing.assert_array_equal(a.bcost, b.bcost)


def test_odd_budget_columns_copy_even_ones():
    """All costs are even (32 + size*{2,4,8}), so column 2k+1 equals column 2k in
    value AND pointers — the GPU stores the budget axis at stride 2 (Q6)."""
    rng = np.random.default_rng(4)
    P = _rand_P(rng, 48, 60)
    res = DP.dp_literal_c(P, 1501, Q.SIZES, Q.TYPES)
    for arr in (res.best, res.btype, res.bsize, res.bcost):
        np.testing.assert_array_equal(arr[:, 1::2], arr[:, 0:-1:2])


def test_scan_form_of_one_pass_equals_literal_loop():
    """Q7: one (i, size) pass of the literal loop equals
    new[b] = old[b] if old[b] <= S[b] else S[b], S = leftmost-argmin prefix scan of
    C[b] = first-min over types of E_t + best[i-size, b-cost_t] (the GPU's form)."""
    rng = np.random.default_rng(5)
    for trial in range(30):
        n, r, B = 16, int(rng.integers(4, 40)), int(rng.integers(50, 600))
        sizes = (1, 2, 4, 16)
        P = _rand_P(rng, n, r)
        if trial % 3 == 0:
            P = np.round(P * 2) / 2                                 # many ties
        Z, Qt = DP.ez_tables(P, sizes, Q.TYPES)
        ref = DP.dp_literal(P, B, sizes, Q.TYPES, ez=(Z, Qt))
        init = DP.canonical_sq_sum(P)
        best = np.full((r + 1, B + 1), init)
        ptr = np.zeros((r + 1, B + 1, 3), dtype=np.int64)
        for i in range(1, r + 1):
            for si, s in enumerate(sizes):
                if s > i:
                    continue
                Cv = np.full(B + 1, np.inf)
                Cp = np.zeros((B + 1, 3), dtype=np.int64)
                for ti, t in enumerate(Q.TYPES):          # first-min over types, P:L1568 order
                    c = Q.cost_bits(s, t)
                    e = -Z[i, si] + Qt[i, si, ti]
                    for b in range(max(1, c), B + 1):
                        v = e + best[i - s, b - c]
                        if v < Cv[b]:
                            Cv[b] = v
                            Cp[b] = (t, s, c)
                Sv, Sp = np.inf, np.zeros(3, dtype=np.int64)
                for b in range(1, B + 1):                  # leftmost-argmin inclusive scan
                    if Cv[b] < Sv:
                        Sv, Sp = Cv[b], Cp[b].copy()
                    if not best[i, b] <= Sv:
                        best[i, b] = Sv
                        ptr[i, b] = Sp
        np.testing.assert_array_equal(best, ref.best)
        np.testing.assert_array_equal(ptr[..., 0], ref.btype)
        np.testing.assert_array_equal(ptr[..., 1], ref.bsize)
        np.testing.assert_array_equal(ptr[..., 2], ref.bcost)


def test_dp_beats_pure_pca_truncation():
    """SPEC acceptance 8 / P:L1345 direction: at equal budget, the DP plan's error
    is <= keeping the leading k = B // 34 PCs exactly (size-1 groups) and dropping
    the rest — that plan is feasible for the DP."""
    rng = np.random.default_rng(6)
    P = _rand_P(rng, 96, 120)
    for B in (68, 340, 1020, 3400):
        res = DP.dp_literal_c(P, B, Q.SIZES, Q.TYPES)
        plan = DP.backtrack(res, B)
        k = min(B // 34, P.shape[1])
        trunc = DP.Plan(r=P.shape[1], blocks=[(j, 1, Q.T_INT2) for j in range(k)])
        assert DP.plan_error(P, plan) <= DP.plan_error(P, trunc) * (1 + 1e-12)


def test_budget_rule():
    assert DP.budget_bits(32768, 16) == 32768           # headline: 4096 B per token per stream
    assert DP.budget_bits(128, 16) == 128
    assert DP.budget_bits(40960, 20) == 32768


def test_vectorised_ez_tables_equal_the_block_loop():
    """ez_tables stacks many blocks per NumPy call; it must reproduce the plain
    per-block loop bit for bit (same expressions, same Q9 summation order)."""
    rng = np.random.default_rng(11)
    for n, r, sizes in ((37, 40, (1, 2, 4)), (100, 130, (1, 16, 64, 256, 1024)), (7, 300, (1, 16, 64, 256))):
        P = rng.standard_normal((n, r)) * (1 + np.arange(r)) ** -0.8
        a = DP.ez_tables_loop(P, sizes)
        b = DP.ez_tables(P, sizes, max_elems=5000)
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(a[1], b[1])
