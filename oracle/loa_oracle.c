/* C restatement of the reference LOA builder -- TEST INFRASTRUCTURE ONLY.
 *
 * Restates /root/reference/pkg/src/rowwin/layout.py:186-263
 * (build_windows_optimized, Algorithm 6 of arXiv 2412.08902) with identical
 * integer semantics, so LOA parity can be checked on graphs far larger than the
 * Python reference finishes in reasonable time.  Only tests/ and bench.py's
 * CPU baseline may call it (see oracle/rowwin_oracle.py header).
 *
 *  - candidates: the first `vw` UNVISITED sorted positions at or after the seed
 *    position (layout.py:112-115, 234); kept as a doubly linked list here
 *    instead of the reference's O(n) flatnonzero rescan -- same set, same order.
 *  - score: (cur_eles + deg) / (cur_cols + deg - cns[v]); den 0 -> (0, 1)
 *    (layout.py:80-91).
 *  - argmax: exact cross multiplication, ties to strictly higher degree, then
 *    earliest scan index (layout.py:118-130).
 *  - admit(v): every column of N(v) not yet in the window increments cns[u] for
 *    u in N(col) (layout.py:211-219); sparse reset at window close (260-262).
 *
 * order: the sort_by_min_neighbor permutation (layout.py:99-109), computed by
 * the caller.  Output: out_order (groups concatenated), gptr (group offsets).
 * Returns the number of groups, or -1 on allocation failure.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

int oracle_loa(const int64_t* rp, const int32_t* ci, int64_t n, int32_t vw, int32_t gs,
               const int64_t* order, int64_t* out_order, int64_t* gptr) {
  int64_t* next = (int64_t*)malloc(sizeof(int64_t) * (n + 2));
  int64_t* prev = (int64_t*)malloc(sizeof(int64_t) * (n + 2));
  int64_t* cns = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  int64_t* stamp = (int64_t*)malloc(sizeof(int64_t) * (n + 1));
  int64_t* touched = NULL;
  int64_t ntouched = 0, cap = 1024;
  int64_t* cand = (int64_t*)malloc(sizeof(int64_t) * (vw > 0 ? vw : 1));
  touched = (int64_t*)malloc(sizeof(int64_t) * cap);
  if (!next || !prev || !cns || !stamp || !cand || !touched) return -1;
  /* linked list over sorted positions 0..n-1 with sentinel n */
  for (int64_t p = 0; p <= n; ++p) { next[p] = p + 1; prev[p] = p - 1; stamp[p] = -1; }
  int64_t head = 0; /* first unvisited position */
  int64_t ngroups = 0, outpos = 0;
  gptr[0] = 0;
#define UNLINK(p) do { int64_t _p = (p); if (prev[_p] >= 0) next[prev[_p]] = next[_p]; else head = next[_p]; \
                       prev[next[_p]] = prev[_p]; } while (0)
  while (head < n) {
    int64_t seed = head; /* smallest unvisited position == next seed (layout.py:222-226) */
    int64_t cur_eles = 0, cur_cols = 0;
    int64_t win = ngroups;
    ntouched = 0;
    int64_t v0 = order[seed];
    UNLINK(seed);
    int64_t glen = 0;
    out_order[outpos + glen++] = v0;
    /* admit(v) */
    int64_t v = v0;
    for (;;) {
      for (int64_t e = rp[v]; e < rp[v + 1]; ++e) {
        int64_t c = ci[e];
        if (stamp[c] == win) continue;
        stamp[c] = win;
        cur_cols++;
        for (int64_t f = rp[c]; f < rp[c + 1]; ++f) {
          int64_t u = ci[f];
          if (cns[u] == 0) {
            if (ntouched == cap) { cap *= 2; touched = (int64_t*)realloc(touched, sizeof(int64_t) * cap); if (!touched) return -1; }
            touched[ntouched++] = u;
          }
          cns[u] += 1;
        }
      }
      cur_eles += rp[v + 1] - rp[v];
      if (glen >= gs) break;
      /* scan: first vw unvisited positions >= seed; seed is visited, so start at head-of-list >= seed */
      int64_t nc = 0;
      int64_t p = head;
      /* every unvisited position is >= seed because seed was the smallest unvisited */
      while (p < n && nc < vw) { cand[nc++] = p; p = next[p]; }
      if (nc == 0) break;
      int64_t bn = 0, bd = 1, bdeg = 0, bp = -1;
      for (int64_t k = 0; k < nc; ++k) {
        int64_t w = order[cand[k]];
        int64_t d = rp[w + 1] - rp[w];
        int64_t num = cur_eles + d;
        int64_t den = cur_cols + d - cns[w];
        if (den == 0) { num = 0; den = 1; }
        if (k == 0) { bn = num; bd = den; bdeg = d; bp = cand[k]; continue; }
        __int128 lhs = (__int128)num * bd, rhs = (__int128)bn * den;
        if (lhs > rhs || (lhs == rhs && d > bdeg)) { bn = num; bd = den; bdeg = d; bp = cand[k]; }
      }
      UNLINK(bp);
      v = order[bp];
      out_order[outpos + glen++] = v;
    }
    outpos += glen;
    ngroups++;
    gptr[ngroups] = outpos;
    for (int64_t t = 0; t < ntouched; ++t) cns[touched[t]] = 0;
  }
#undef UNLINK
  free(next); free(prev); free(cns); free(stamp); free(cand); free(touched);
  return (int)ngroups;
}
