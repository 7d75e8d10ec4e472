/* KVTC oracle — TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * The loop nest of the paper's "Dynamic Programming Precision Assignment"
 * pseudocode, written out literally in plain C for
 * instances too large for the Python loop (oracle/dp.py::dp_literal).  The
 * per-(i, size, type) error change E = -sum(x*x) + sum((x-x^)^2) is computed by
 * the Python oracle (oracle/dp.py::ez_tables) and passed in; this file only
 * runs the table recursion:
 *
 *   best[i][b] = init for all i, b                                  (L1553-1557)
 *   for i in 1..r, for size in sizes (size <= i), for b in 1..B:    (L1570-1575)
 *     if best[i][b] > best[i][b-1]: copy value and pointers          (L1576-1580)
 *     for t in types: if cost(size,t) <= b:                          (L1582-1587)
 *        cand = E[i][size][t] + best[i-size][b-cost]                 (L1592-1594)
 *        if best[i][b] > cand: take it                               (L1594-1598)
 *
 * Compiled with -ffp-contract=off; every operation is one IEEE fp64 add.
 * Pinned to the Python loop in tests/test_oracle_dp.py.
 */
#include <stdint.h>

int kvtc_oracle_dp(int r, int B, int nsizes, const int32_t *sizes, int ntypes,
                   const int32_t *types, const int32_t *type_bits,
                   const double *E, /* [(r+1) * nsizes * ntypes] */
                   double init, double *best, int32_t *btype, int32_t *bsize,
                   int32_t *bcost) {
  const long W = (long)B + 1;
  for (long k = 0; k < (long)(r + 1) * W; ++k) {
    best[k] = init;
    btype[k] = 0;
    bsize[k] = 0;
    bcost[k] = 0;
  }
  for (int i = 1; i <= r; ++i) {
    for (int si = 0; si < nsizes; ++si) {
      const int s = sizes[si];
      if (s > i) continue;
      double *row = best + (long)i * W;
      const double *prev = best + (long)(i - s) * W;
      int32_t *rt = btype + (long)i * W, *rs = bsize + (long)i * W, *rc = bcost + (long)i * W;
      for (int b = 1; b <= B; ++b) {
        if (row[b] > row[b - 1]) {
          row[b] = row[b - 1];
          rt[b] = rt[b - 1];
          rs[b] = rs[b - 1];
          rc[b] = rc[b - 1];
        }
        for (int ti = 0; ti < ntypes; ++ti) {
          const int used = type_bits[ti] == 0 ? 0 : s * type_bits[ti] + 32;
          if (used <= b) {
            const double change = E[((long)i * nsizes + si) * ntypes + ti];
            const double cand = change + prev[b - used];
            if (row[b] > cand) {
              row[b] = cand;
              rt[b] = types[ti];
              rs[b] = s;
              rc[b] = used;
            }
          }
        }
      }
    }
  }
  return 0;
}
