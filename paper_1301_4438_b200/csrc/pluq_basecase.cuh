// Algorithm 2 (Z-curve iterative PLUQ) as a CTA-cooperative device routine.
//
// Restates /root/reference/pkg/src/pluq/iterative.py:30-93 with LAZY rotations:
// the elimination runs in the block's original coordinates and a single
// gather at the end realises every order-preserving row/column rotation.
// Equivalence (checked bit-for-bit against the reference goldens by the oracle,
// oracle/pluq_oracle.py:basecase): rotations keep non-pivot rows/columns in
// original relative order, so (a) "rows after the pivot row" are the non-pivot
// rows with a larger original index, (b) the frontier row i / column j is still
// the untouched original row i / column j, and (c) the segment A[r:i, j] is the
// non-pivot rows among the first i originals.
//
// The routine works on a generic pointer: the batch/small-node kernel passes
// shared memory, the large-block kernel passes global memory.
#pragma once
#include "pluq_common.cuh"

namespace pluq {

struct BcShared {
  int i, j, r, found, pr, pc, done;
  int minv;
  unsigned long long below, right;
};

// CTA-wide minimum of `v` (INT_MAX = none). Uses sh->minv; ends synchronized.
__device__ __forceinline__ int cta_min(int v, BcShared* sh) {
  if (threadIdx.x == 0) sh->minv = 0x7fffffff;
  __syncthreads();
  int w = __reduce_min_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0 && w != 0x7fffffff) atomicMin(&sh->minv, w);
  __syncthreads();
  int res = sh->minv;
  __syncthreads();
  return res;
}

// Scratch the base case needs (all of length >= m or n as noted); generic pointers.
struct BcScratch {
  uint8_t* prow;   // m
  uint8_t* pcol;   // n
  int* rord;       // min(m,n)
  int* cord;       // min(m,n)
  int* rowat;      // m
  int* colat;      // n
};

// Warp-0 Z-curve search while both frontiers are interior (iterative.py:36-57).
// Returns with sh->found / sh->pr / sh->pc / sh->i / sh->j updated.
__device__ __forceinline__ void bc_search_interior(const View& x, const BcScratch& s, BcShared* sh) {
  const int lane = threadIdx.x & 31;
  int i = sh->i, j = sh->j;
  const int m = x.m, n = x.n;
  int found = 0, pr = -1, pc = -1;
  while (i < m && j < n) {
    // column segment A[r:i, j]: first non-pivot original row < i
    for (int base = 0; base < i; base += 32) {
      int rho = base + lane;
      bool pred = rho < i && !s.prow[rho] && x.at(rho, j) != 0u;
      unsigned b = __ballot_sync(0xffffffffu, pred);
      if (b) { pr = base + __ffs(b) - 1; pc = j; found = 1; break; }
    }
    if (found) { j += 1; break; }
    // row segment A[i, r:j]: first non-pivot original column < j
    for (int base = 0; base < j; base += 32) {
      int gam = base + lane;
      bool pred = gam < j && !s.pcol[gam] && x.at(i, gam) != 0u;
      unsigned b = __ballot_sync(0xffffffffu, pred);
      if (b) { pr = i; pc = base + __ffs(b) - 1; found = 1; break; }
    }
    if (found) { i += 1; break; }
    if (x.at(i, j) != 0u) { pr = i; pc = j; found = 1; i += 1; j += 1; break; }
    i = min(i + 1, m);
    j = min(j + 1, n);
  }
  if (lane == 0) { sh->i = i; sh->j = j; sh->found = found; sh->pr = pr; sh->pc = pc; }
}

// Base case on view x. Writes P.sigma (psig, length m) and Q.sigma (qsig, length n),
// returns the rank.  `cnt` is only touched by thread 0.  `gather` is called to
// apply the final row / column gathers (memory-space specific).
template <class Gather>
__device__ int basecase_cta(const View& x, int* psig, int* qsig, const BcScratch& s, BcShared* sh,
                            const ModP& mp, Counts* cnt, Gather&& gather) {
  const int m = x.m, n = x.n;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  for (int q = tid; q < m; q += nt) s.prow[q] = 0;
  for (int q = tid; q < n; q += nt) s.pcol[q] = 0;
  if (tid == 0) { sh->i = 0; sh->j = 0; sh->r = 0; sh->done = 0; }
  __syncthreads();
  while (true) {
    int i = sh->i, j = sh->j;
    __syncthreads();  // every thread has read the frontier before warp 0 may move it
    int pr = -1, pc = -1;
    if (i < m && j < n) {
      if (warp == 0) bc_search_interior(x, s, sh);
      __syncthreads();
      if (!sh->found) continue;  // frontier reached a border; re-dispatch
      pr = sh->pr; pc = sh->pc;
    } else if (j < n) {
      // i == m: column segment spans every non-pivot row; first column >= j with a nonzero
      int best = 0x7fffffff;
      for (int base = j; base < n && best == 0x7fffffff; base += nt) {
        int col = base + tid;
        int hit = 0x7fffffff;
        if (col < n)
          for (int rho = 0; rho < m; ++rho)
            if (!s.prow[rho] && x.at(rho, col) != 0u) { hit = col; break; }
        best = cta_min(hit, sh);
      }
      if (best == 0x7fffffff) break;
      int hit = 0x7fffffff;
      for (int rho = tid; rho < m; rho += nt)
        if (!s.prow[rho] && x.at(rho, best) != 0u) { hit = rho; break; }
      pr = cta_min(hit, sh);
      pc = best;
      if (tid == 0) sh->j = best + 1;
    } else if (i < m) {
      // j == n: row segment spans every non-pivot column; first row >= i with a nonzero
      int best = 0x7fffffff;
      for (int base = i; base < m && best == 0x7fffffff; base += nt) {
        int rw = base + tid;
        int hit = 0x7fffffff;
        if (rw < m)
          for (int gam = 0; gam < n; ++gam)
            if (!s.pcol[gam] && x.at(rw, gam) != 0u) { hit = rw; break; }
        best = cta_min(hit, sh);
      }
      if (best == 0x7fffffff) break;
      int hit = 0x7fffffff;
      for (int gam = tid; gam < n; gam += nt)
        if (!s.pcol[gam] && x.at(best, gam) != 0u) { hit = gam; break; }
      pc = cta_min(hit, sh);
      pr = best;
      if (tid == 0) sh->i = best + 1;
    } else {
      break;
    }
    // ---- elimination below/right of the pivot (iterative.py:59-75) ----
    const uint32_t inv = invmod(x.at(pr, pc), mp);
    const uint32_t* prow_ptr = x.row(pr);
    for (int rho = pr + 1 + warp; rho < m; rho += nw) {
      if (s.prow[rho]) continue;
      uint32_t* rp = x.row(rho);
      uint32_t a = rp[pc];
      if (a == 0u) continue;
      uint32_t mult = mulmod(a, inv, mp);
      __syncwarp();
      if (lane == 0) rp[pc] = mult;
      for (int gam = pc + 1 + lane; gam < n; gam += 32) {
        if (s.pcol[gam]) continue;
        uint32_t b = prow_ptr[gam];
        if (b) rp[gam] = submod(rp[gam], mulmod(mult, b, mp), mp);
      }
    }
    if (tid == 0) {
      // reference charges: below = rows after the pivot in current order, right = cols after
      int r = sh->r;
      long long below = m - 1 - pr, right = n - 1 - pc;
      for (int t = 0; t < r; ++t) { below -= (s.rord[t] > pr); right -= (s.cord[t] > pc); }
      if (below > 0) {
        cnt->inv += 1; cnt->mul += below; cnt->red += below;
        if (right > 0) {
          cnt->mul += below * right; cnt->add += below * right; cnt->red += below * right;
        }
      }
    }
    __syncthreads();
    if (tid == 0) {
      int r = sh->r;
      s.prow[pr] = 1; s.pcol[pc] = 1; s.rord[r] = pr; s.cord[r] = pc; sh->r = r + 1;
    }
    __syncthreads();
  }
  __syncthreads();
  const int r = sh->r;
  // final positions: pivots first (in pivot order), then non-pivots in original order
  for (int t = tid; t < r; t += nt) { s.rowat[t] = s.rord[t]; s.colat[t] = s.cord[t]; }
  for (int q = tid; q < m; q += nt) {
    if (s.prow[q]) continue;
    int before = 0;
    for (int t = 0; t < r; ++t) before += (s.rord[t] < q);
    s.rowat[r + q - before] = q;
  }
  for (int q = tid; q < n; q += nt) {
    if (s.pcol[q]) continue;
    int before = 0;
    for (int t = 0; t < r; ++t) before += (s.cord[t] < q);
    s.colat[r + q - before] = q;
  }
  __syncthreads();
  for (int t = tid; t < m; t += nt) psig[s.rowat[t]] = t;  // P.sigma = inverse(row_at)
  for (int t = tid; t < n; t += nt) qsig[t] = s.colat[t];   // Q.sigma = col_at
  __syncthreads();
  gather(s.rowat, s.colat, r);
  __syncthreads();
  return r;
}

}  // namespace pluq
