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
__device__ __forceinline__ void bc_search_interior(const View x, const BcScratch s, BcShared* sh) {
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
__device__ int basecase_cta(const View x, int* psig, int* qsig, const BcScratch s, BcShared* sh,
                            const ModP mp, Counts* cnt, Gather&& gather) {
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

// ------------------------------------------------------------------------------------
// Single-warp base case (shared-memory blocks inside the small-node kernel).
//
// Same algorithm as basecase_cta, executed by ONE converged warp with __syncwarp
// only: ballots for the Z-curve search, lanes over columns for the rank-1 update,
// and the pivot inverse from a table when p < 2^16 (one load instead of Euclid).
// Called by warp 0 while the other warps of the CTA wait at the next barrier.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t pivot_inverse(uint32_t a, const ModP mp, const uint16_t* tab) {
  return tab ? (uint32_t)tab[a] : invmod(a, mp);
}

// In-place row / column gathers by one warp (cycle walks; lane 0 builds the cycles).
__device__ __forceinline__ void warp_gather(const View v, const int* g, bool rows, int* seq, int* lens,
                                            int* mark) {
  const int lane = threadIdx.x & 31;
  const int len_total = rows ? v.m : v.n;
  bool ident = true;
  for (int t = lane; t < len_total; t += 32) ident &= (g[t] == t);
  if (__all_sync(0xffffffffu, ident)) return;
  int nc = 0;
  if (lane == 0) {
    for (int t = 0; t < len_total; ++t) mark[t] = 0;
    int pos = 0;
    for (int s0 = 0; s0 < len_total; ++s0) {
      if (mark[s0] || g[s0] == s0) continue;
      int cur = s0, len = 0;
      do { seq[pos++] = cur; mark[cur] = 1; cur = g[cur]; ++len; } while (cur != s0);
      lens[nc++] = len;
    }
  }
  nc = __shfl_sync(0xffffffffu, nc, 0);
  __syncwarp();
  const int other = rows ? v.n : v.m;
  for (int o = lane; o < other; o += 32) {
    int pos = 0;
    for (int cy = 0; cy < nc; ++cy) {
      const int len = lens[cy];
      if (rows) {
        uint32_t tmp = v.at(seq[pos], o);
        for (int q = 0; q + 1 < len; ++q) v.at(seq[pos + q], o) = v.at(seq[pos + q + 1], o);
        v.at(seq[pos + len - 1], o) = tmp;
      } else {
        uint32_t* row = v.row(o);
        uint32_t tmp = row[seq[pos]];
        for (int q = 0; q + 1 < len; ++q) row[seq[pos + q]] = row[seq[pos + q + 1]];
        row[seq[pos + len - 1]] = tmp;
      }
      pos += len;
    }
  }
  __syncwarp();
}

// Returns the rank; psig/qsig receive P.sigma / Q.sigma; `scale` needs m words.
//
// FRACTION-FREE elimination: every row rho carries a scale S[rho] (stored = S * true).
// Pivot (pr, pc) with stored value a: each later non-pivot row with b = A[rho][pc] != 0
// becomes  A[rho][g] = a*A[rho][g] - b*A[pr][g]  on the non-pivot columns right of pc,
// A[rho][pc] = b*S[pr] (the L entry, in row-scale units) and a*A[rho][g] elsewhere, with
// S[rho] *= a.  Zero tests are unchanged (S != 0), so the pivot sequence is exactly
// the reference's; no inverse sits on the per-pivot chain.  At the end every row is
// multiplied by S^-1 (inverses computed in parallel, one per row), which yields the
// reference's normalised L \ U values bit for bit.
//
// Warp 0 runs the Z-curve search (ballots); the whole CTA updates the rows below the
// pivot (read phase / barrier / write phase), so the per-pivot latency is one round of
// loads + two multiplications regardless of the block height.
template <class Gather>
__device__ int basecase_ff(const View x, int* psig, int* qsig, const BcScratch s, uint32_t* scale, uint32_t* bcol,
                           BcShared* sh, const ModP mp, const uint16_t* invtab, Counts* cnt, Gather&& gather) {
  const int m = x.m, n = x.n;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const unsigned FULL = 0xffffffffu;
  uint32_t* __restrict__ A = x.a;
  const int64_t ld = x.ld;
  uint8_t* __restrict__ prow = s.prow;
  uint8_t* __restrict__ pcol = s.pcol;
  int* __restrict__ rord = s.rord;
  int* __restrict__ cord = s.cord;
  uint32_t* __restrict__ S = scale;
  for (int q = tid; q < m; q += nt) { prow[q] = 0; S[q] = 1; }
  for (int q = tid; q < n; q += nt) pcol[q] = 0;
  __syncthreads();
  int r = 0, i = 0, j = 0;  // meaningful in warp 0
  unsigned long long c_mul = 0, c_add = 0, c_inv = 0, c_red = 0;
  // update layout for n <= nt: C column lanes (power of two >= n) x R rows in flight
  int C = 1;
  while (C < n && C < nt) C <<= 1;
  const int R = nt / C, tc = tid & (C - 1), tr = tid / C;
  while (true) {
    if (warp == 0) {
      __syncwarp();
      int pr = -1, pc = -1;
      // ---------------- Z-curve pivot search (iterative.py:36-57) ----------------
      while (pr < 0) {
        if (i < m && j < n) {
          for (int base = 0; base < i && pr < 0; base += 32) {
            const int rho = base + lane;
            const unsigned bb = __ballot_sync(FULL, rho < i && !prow[rho] && A[rho * ld + j] != 0u);
            if (bb) { pr = base + __ffs(bb) - 1; pc = j; }
          }
          if (pr >= 0) { j += 1; break; }
          for (int base = 0; base < j && pr < 0; base += 32) {
            const int gam = base + lane;
            const unsigned bb = __ballot_sync(FULL, gam < j && !pcol[gam] && A[i * ld + gam] != 0u);
            if (bb) { pr = i; pc = base + __ffs(bb) - 1; }
          }
          if (pr >= 0) { i += 1; break; }
          if (A[i * ld + j] != 0u) { pr = i; pc = j; i += 1; j += 1; break; }
          i = min(i + 1, m);
          j = min(j + 1, n);
        } else if (j < n) {
          int best = -1;  // i == m: first column >= j with a nonzero in a non-pivot row
          for (int base = j; base < n && best < 0; base += 32) {
            const int col = base + lane;
            bool hit = false;
            if (col < n)
              for (int rho = 0; rho < m && !hit; ++rho) hit = !prow[rho] && A[rho * ld + col] != 0u;
            const unsigned bb = __ballot_sync(FULL, hit);
            if (bb) best = base + __ffs(bb) - 1;
          }
          if (best < 0) { j = n; break; }
          for (int base = 0; base < m && pr < 0; base += 32) {
            const int rho = base + lane;
            const unsigned bb = __ballot_sync(FULL, rho < m && !prow[rho] && A[rho * ld + best] != 0u);
            if (bb) pr = base + __ffs(bb) - 1;
          }
          pc = best;
          j = best + 1;
        } else if (i < m) {
          int best = -1;  // j == n: first row >= i with a nonzero in a non-pivot column
          for (int base = i; base < m && best < 0; base += 32) {
            const int rw = base + lane;
            bool hit = false;
            if (rw < m)
              for (int gam = 0; gam < n && !hit; ++gam) hit = !pcol[gam] && A[rw * ld + gam] != 0u;
            const unsigned bb = __ballot_sync(FULL, hit);
            if (bb) best = base + __ffs(bb) - 1;
          }
          if (best < 0) { i = m; break; }
          for (int base = 0; base < n && pc < 0; base += 32) {
            const int gam = base + lane;
            const unsigned bb = __ballot_sync(FULL, gam < n && !pcol[gam] && A[best * ld + gam] != 0u);
            if (bb) pc = base + __ffs(bb) - 1;
          }
          pr = best;
          i = best + 1;
        } else {
          break;
        }
      }
      if (pr >= 0) {
        // reference charges (iterative.py:63-75): below / right in the current layout
        int below = 0, right = 0;
        for (int base = pr + 1; base < m; base += 32)
          below += __popc(__ballot_sync(FULL, base + lane < m && !prow[base + lane]));
        for (int base = pc + 1; base < n; base += 32)
          right += __popc(__ballot_sync(FULL, base + lane < n && !pcol[base + lane]));
        if (below > 0) {
          c_inv += 1; c_mul += below; c_red += below;
          const unsigned long long br = (unsigned long long)below * right;
          c_mul += br; c_add += br; c_red += br;
        }
      }
      if (pr >= 0)  // snapshot of the pivot column (rows straddling update chunks read it)
        for (int rho = pr + 1 + lane; rho < m; rho += 32) bcol[rho] = prow[rho] ? 0u : A[rho * ld + pc];
      if (lane == 0) { sh->pr = pr; sh->pc = pc; }
    }
    __syncthreads();
    const int pr = sh->pr, pc = sh->pc;
    if (pr < 0) break;
    // ---------------- fraction-free elimination over the whole CTA ----------------
    const uint32_t a = A[pr * ld + pc];
    const uint32_t spr = S[pr];
    const uint32_t* __restrict__ prw = A + pr * ld;
    // every element is read and written by the same thread (only the bcol snapshot, the
    // untouched pivot row and the flags are shared), so no read/write phase split
    if (n <= nt) {
      for (int rho = pr + 1 + tr; rho < m; rho += R) {
        const uint32_t b = bcol[rho];
        if (!b || tc >= n) continue;
        uint32_t* row = A + rho * ld;
        const int g = tc;
        const uint32_t v = row[g];
        uint32_t w;
        if (g == pc) { w = mulmod(b, spr, mp); S[rho] = mulmod(S[rho], a, mp); }
        else if (g > pc && !pcol[g]) w = submod(mulmod(a, v, mp), mulmod(b, prw[g], mp), mp);
        else w = mulmod(a, v, mp);
        row[g] = w;
      }
    } else {
      for (int rho = pr + 1; rho < m; ++rho) {
        const uint32_t b = bcol[rho];
        if (!b) continue;
        uint32_t* row = A + rho * ld;
        for (int g = tid; g < n; g += nt) {
          const uint32_t v = row[g];
          uint32_t w;
          if (g == pc) { w = mulmod(b, spr, mp); S[rho] = mulmod(S[rho], a, mp); }
          else if (g > pc && !pcol[g]) w = submod(mulmod(a, v, mp), mulmod(b, prw[g], mp), mp);
          else w = mulmod(a, v, mp);
          row[g] = w;
        }
      }
    }
    __syncthreads();
    if (tid == 0) { prow[pr] = 1; pcol[pc] = 1; rord[r] = pr; cord[r] = pc; }
    ++r;
  }
  if (tid == 0) {
    cnt->mul += c_mul; cnt->add += c_add; cnt->inv += c_inv; cnt->red += c_red;
    sh->r = r;
  }
  // ---- normalise: row rho *= S[rho]^-1 (inverses in parallel) ----
  for (int q = tid; q < m; q += nt) {
    const uint32_t sv = S[q];
    S[q] = sv == 1u ? 1u : pivot_inverse(sv, mp, invtab);
  }
  __syncthreads();
  const int rr = sh->r;
  for (int rho = tid / C; rho < m; rho += R) {
    const uint32_t iv = S[rho];
    if (iv == 1u) continue;
    for (int g = tc; g < n; g += C) A[rho * ld + g] = mulmod(A[rho * ld + g], iv, mp);
  }
  // final positions: pivots first, then the non-pivots in original order
  for (int t = tid; t < rr; t += nt) { s.rowat[t] = rord[t]; s.colat[t] = cord[t]; }
  for (int q = tid; q < m; q += nt) {
    if (prow[q]) continue;
    int before = 0;
    for (int t = 0; t < rr; ++t) before += (rord[t] < q);
    s.rowat[rr + q - before] = q;
  }
  for (int q = tid; q < n; q += nt) {
    if (pcol[q]) continue;
    int before = 0;
    for (int t = 0; t < rr; ++t) before += (cord[t] < q);
    s.colat[rr + q - before] = q;
  }
  __syncthreads();
  for (int t = tid; t < m; t += nt) psig[s.rowat[t]] = t;
  for (int t = tid; t < n; t += nt) qsig[t] = s.colat[t];
  __syncthreads();
  gather(s.rowat, s.colat, rr);
  __syncthreads();
  return rr;
}

}  // namespace pluq
