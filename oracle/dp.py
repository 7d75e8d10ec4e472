"""DP bit allocation — oracle (test infrastructure).

Follows the pseudocode of P:L1541-1603 ("Dynamic Programming Precision
Assignment") literally, in its loop order and with its strict ``>`` tests:

  best_error[i, b] initialised to ||P||_F^2 for all (i, b)
  for i in 1..r: for block_size in [1,16,64,256,1024] (<= i):
    for budget in 1..B:
      if best[i,b] > best[i,b-1]: copy (value, type, size, cost)
      for t in [None, int2, int4, fp8]:
        x^, used = simulate_quantization(P[:, i-size:i], t)
        if used <= b:
          change = -sum(x*x) + sum((x - x^)^2)
          if best[i,b] > change + best[i-size, b-used]: take it

The quantisation simulation of one block depends only on (i, size, t), so it
is evaluated once per (i, size, t) (``ez_tables``) instead of once per budget:
the same fp64 value, hoisted.  Sums use the canonical order of reading Q9
(per row: sequential over the block's columns, each product rounded then
added; across rows: an adjacent-pair binary tree over the rows zero-padded to a
power of two) — the paper is silent on summation order, and the GPU uses the
same tree so the plan can be bit-exact.

Budget (Q6): B = floor(feature_bits * p_original / CR).
Backtracking (Q7): from (r, B) emit (size, type) at (i, b) and move to
(i - size, b - cost) until size == 0 or i == 0; PCs not covered are None.

Pins (tests/test_oracle_dp.py): exact equality with brute-force enumeration on
random tiny instances (the proof-by-induction claim of P:L1604-1610 made
executable), the base case best[0,:] = best[:,0] = ||P||^2,
monotonicity in b, plan cost <= B, plan error re-simulated == table value.
The C loop (oracle/dp_literal.c) is pinned to the Python loop.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

from .quant import BITS, SIZES, TYPES, T_NONE, cost_bits, simulate_quantization


# ----------------------------------------------------------- canonical sums (Q9)
def tree_sum(v) -> float:
    """Adjacent-pair binary tree over v zero-padded to a power of two."""
    v = np.asarray(v, dtype=np.float64)
    n = max(1, len(v))
    k = 1
    while k < n:
        k *= 2
    w = np.zeros(k)
    w[: len(v)] = v
    while len(w) > 1:
        w = w[0::2] + w[1::2]
    return float(w[0])


def row_sq_sums(e) -> np.ndarray:
    """Per row: s = 0; for each column c in order: s = s + e[:, c]*e[:, c]."""
    e = np.asarray(e, dtype=np.float64)
    s = np.zeros(e.shape[:-1])
    for c in range(e.shape[-1]):
        s = s + e[..., c] * e[..., c]
    return s


def canonical_sq_sum(e) -> float:
    return tree_sum(row_sq_sums(e))


# ------------------------------------------------------------------- E/Z tables
def ez_tables_loop(P, sizes=SIZES, types=TYPES):
    """Z[i, si] = sum x^2 and Q[i, si, ti] = sum (x - x^)^2 over P[:, i-size:i],
    one block at a time (the plain form; ``ez_tables`` evaluates the same
    expressions for many blocks per NumPy call).  Rows i = 0..r (row 0 unused);
    NaN where size > i."""
    P = np.asarray(P, dtype=np.float64)
    n, r = P.shape
    Z = np.full((r + 1, len(sizes)), np.nan)
    Q = np.full((r + 1, len(sizes), len(types)), np.nan)
    for si, s in enumerate(sizes):
        for i in range(s, r + 1):
            blk = P[:, i - s:i]
            Z[i, si] = canonical_sq_sum(blk)
            for ti, t in enumerate(types):
                xh, _ = simulate_quantization(blk, t)
                Q[i, si, ti] = canonical_sq_sum(blk - xh)
    return Z, Q


def _tree_sum_rows(v):
    """tree_sum applied to every column of v [n, k] (rows zero-padded to a
    power of two, adjacent pairs added level by level)."""
    n = v.shape[0]
    k = 1
    while k < n:
        k *= 2
    w = np.zeros((k,) + v.shape[1:])
    w[:n] = v
    while w.shape[0] > 1:
        w = w[0::2] + w[1::2]
    return w[0]


def ez_tables(P, sizes=SIZES, types=TYPES, max_elems: int = 1 << 23):
    """Same values as ``ez_tables_loop``, bit for bit: every block's quantisation
    is per row (Q1), so many blocks are stacked as extra rows of one
    ``quantize_rows`` call; the sums keep the canonical order of Q9 (per row
    sequential over the block's columns, product then add; across rows the
    adjacent-pair tree).  Needed for the DP parity at production shape
    (r ~ 2000+ PCs with 256- and 1024-blocks)."""
    P = np.asarray(P, dtype=np.float64)
    n, r = P.shape
    Z = np.full((r + 1, len(sizes)), np.nan)
    Q = np.full((r + 1, len(sizes), len(types)), np.nan)
    for si, s in enumerate(sizes):
        if s > r:
            continue
        ends = np.arange(s, r + 1)
        step = max(1, max_elems // (n * s))
        for c0 in range(0, len(ends), step):
            e = ends[c0:c0 + step]
            nb = len(e)
            # blk[row, b, col] = P[row, e[b] - s + col]
            blk = np.lib.stride_tricks.sliding_window_view(P, s, axis=1)[:, e - s, :]
            Z[e, si] = _tree_sum_rows(row_sq_sums(blk))
            flat = blk.reshape(n * nb, s)
            for ti, t in enumerate(types):
                xh, _ = simulate_quantization(flat, t)
                Q[e, si, ti] = _tree_sum_rows(row_sq_sums((flat - xh).reshape(n, nb, s)))
    return Z, Q


@dataclass
class DPResult:
    best: np.ndarray          # (r+1, B+1) fp64
    btype: np.ndarray         # (r+1, B+1) int  type code (P:L1568 order)
    bsize: np.ndarray         # (r+1, B+1) int  block size (0 = no decision)
    bcost: np.ndarray         # (r+1, B+1) int  bit cost
    init: float
    sizes: tuple = SIZES
    types: tuple = TYPES


def dp_literal(P, B: int, sizes=SIZES, types=TYPES, ez=None) -> DPResult:
    """The pseudocode's loop nest, in Python (for small instances)."""
    P = np.asarray(P, dtype=np.float64)
    n, r = P.shape
    Z, Q = ez if ez is not None else ez_tables(P, sizes, types)
    init = canonical_sq_sum(P)
    best = np.full((r + 1, B + 1), init)
    btype = np.zeros((r + 1, B + 1), dtype=np.int64)
    bsize = np.zeros((r + 1, B + 1), dtype=np.int64)
    bcost = np.zeros((r + 1, B + 1), dtype=np.int64)
    for i in range(1, r + 1):
        for si, s in enumerate(sizes):
            if s > i:
                continue
            changes = [(t, cost_bits(s, t), -Z[i, si] + Q[i, si, ti]) for ti, t in enumerate(types)]
            for b in range(1, B + 1):
                if best[i, b] > best[i, b - 1]:
                    best[i, b] = best[i, b - 1]
                    btype[i, b] = btype[i, b - 1]
                    bsize[i, b] = bsize[i, b - 1]
                    bcost[i, b] = bcost[i, b - 1]
                for t, used, change in changes:
                    if used <= b:
                        cand = change + best[i - s, b - used]
                        if best[i, b] > cand:
                            best[i, b] = cand
                            btype[i, b] = t
                            bsize[i, b] = s
                            bcost[i, b] = used
    return DPResult(best, btype, bsize, bcost, init, tuple(sizes), tuple(types))


_LIB = None


def _c_lib():
    global _LIB
    if _LIB is None:
        here = os.path.dirname(os.path.abspath(__file__))
        so = os.path.join(here, "_dp_literal.so")
        src = os.path.join(here, "dp_literal.c")
        if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
            build_c()
        _LIB = ctypes.CDLL(so)
        _LIB.kvtc_oracle_dp.restype = ctypes.c_int
    return _LIB


def build_c() -> str:
    """Compile oracle/dp_literal.c (plain C, gcc) — the checker, not the product."""
    import subprocess
    here = os.path.dirname(os.path.abspath(__file__))
    so = os.path.join(here, "_dp_literal.so")
    subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared",
                           "-o", so, os.path.join(here, "dp_literal.c")])
    return so


def dp_literal_c(P, B: int, sizes=SIZES, types=TYPES, ez=None) -> DPResult:
    """Same loop nest in plain C (oracle/dp_literal.c), for larger instances."""
    P = np.asarray(P, dtype=np.float64)
    n, r = P.shape
    Z, Q = ez if ez is not None else ez_tables(P, sizes, types)
    init = canonical_sq_sum(P)
    E = np.zeros((r + 1, len(sizes), len(types)))
    for si in range(len(sizes)):
        for ti in range(len(types)):
            E[:, si, ti] = -Z[:, si] + Q[:, si, ti]
    E = np.ascontiguousarray(np.nan_to_num(E, nan=0.0))
    best = np.empty((r + 1, B + 1))
    btype = np.empty((r + 1, B + 1), dtype=np.int32)
    bsize = np.empty((r + 1, B + 1), dtype=np.int32)
    bcost = np.empty((r + 1, B + 1), dtype=np.int32)
    sz = np.asarray(sizes, dtype=np.int32)
    tp = np.asarray(types, dtype=np.int32)
    tb = np.asarray([BITS[t] for t in types], dtype=np.int32)
    dp = ctypes.POINTER(ctypes.c_double)
    ip = ctypes.POINTER(ctypes.c_int32)
    rc = _c_lib().kvtc_oracle_dp(
        ctypes.c_int(r), ctypes.c_int(B), ctypes.c_int(len(sizes)), sz.ctypes.data_as(ip),
        ctypes.c_int(len(types)), tp.ctypes.data_as(ip), tb.ctypes.data_as(ip),
        E.ctypes.data_as(dp), ctypes.c_double(init), best.ctypes.data_as(dp),
        btype.ctypes.data_as(ip), bsize.ctypes.data_as(ip), bcost.ctypes.data_as(ip))
    assert rc == 0
    return DPResult(best, btype.astype(np.int64), bsize.astype(np.int64),
                    bcost.astype(np.int64), init, tuple(sizes), tuple(types))


# ------------------------------------------------------------------- the plan
@dataclass
class Plan:
    """Contiguous groups over PCs [0, r): (start, size, type); None groups
    included.  ``groups`` lists only the non-None ones in PC order."""
    r: int
    blocks: list = field(default_factory=list)     # [(start, size, type)] covering chosen span

    @property
    def groups(self):
        return [(s, z, t) for (s, z, t) in self.blocks if t != T_NONE]

    @property
    def bits_per_token(self) -> int:
        return sum(cost_bits(z, t) for (_, z, t) in self.groups)

    @property
    def r_eff(self) -> int:
        g = self.groups
        return (g[-1][0] + g[-1][1]) if g else 0


def backtrack(res: DPResult, B: int) -> Plan:
    r = res.best.shape[0] - 1
    i, b = r, B
    blocks = []
    while i > 0:
        s = int(res.bsize[i, b])
        if s == 0:
            break
        t = int(res.btype[i, b])
        c = int(res.bcost[i, b])
        blocks.append((i - s, s, t))
        i -= s
        b -= c
    blocks.reverse()
    return Plan(r=r, blocks=blocks)


def budget_bits(p_original: int, target_cr: float, feature_bits: int = 16) -> int:
    """Q6: B = floor(feature_bits * p / CR) bits per token per stream."""
    return int(np.floor(feature_bits * p_original / target_cr))


def allocate(P, target_cr: float, p_original: int, sizes=SIZES, types=TYPES,
             feature_bits: int = 16, use_c: bool = True):
    """P:L1541-1603 end to end: tables, DP at B, backtrack."""
    B = budget_bits(p_original, target_cr, feature_bits)
    fn = dp_literal_c if use_c else dp_literal
    res = fn(P, B, sizes, types)
    return backtrack(res, B), res, B


def plan_error(P, plan: Plan) -> float:
    """||D - D^q||_F^2 re-simulated group by group."""
    P = np.asarray(P, dtype=np.float64)
    err = P.copy()
    for (s, z, t) in plan.groups:
        xh, _ = simulate_quantization(P[:, s:s + z], t)
        err[:, s:s + z] = P[:, s:s + z] - xh
    return float(np.sum(err * err))


# --------------------------------------------------------------- brute force
def brute_force(P, B: int, sizes, types):
    """Enumerate every covering of PCs [0, r) by blocks (size in ``sizes``,
    type in ``types``) whose cost fits B; value folded exactly as the DP folds
    it: v = init; for each block left to right: v = (Q - Z) + v.  Returns
    (min value, a minimising block list).  Exponential: tiny r only."""
    P = np.asarray(P, dtype=np.float64)
    n, r = P.shape
    Z, Q = ez_tables(P, sizes, types)
    init = canonical_sq_sum(P)
    best = [np.inf, None]

    def rec(i, used, val, path):
        if i == r:
            if val < best[0]:
                best[0], best[1] = val, list(path)
            return
        for si, s in enumerate(sizes):
            j = i + s
            if j > r:
                continue
            for ti, t in enumerate(types):
                c = cost_bits(s, t)
                if used + c > B:
                    continue
                change = -Z[j, si] + Q[j, si, ti]
                path.append((i, s, t))
                rec(j, used + c, change + val, path)
                path.pop()

    rec(0, 0, init, [])
    return best[0], best[1]
