// Whole-node PLUQ inside one CTA, with the block resident in shared memory.
//
// This is Algorithm 1 (/root/reference/pkg/src/pluq/recursive.py:186-256) run
// cooperatively by one CTA: same split (m//2, n//2), same terminal tests, same
// 12 block permutations / 6 TRSM / 6 MM calls, same S/T block permutations and
// P/Q composition.  It serves (a) the batched API (one CTA per independent
// matrix, BASELINE cfg2) and (b) every node of the large-matrix recursion that
// fits in shared memory, so the host driver never walks the small nodes.
//
// Shared-memory layout: the block with an odd row pitch (bank-conflict free
// column walks) followed by a bump "stack" of int32 words.  Every thread runs
// the same control flow and derives identical stack offsets, so allocation
// needs no synchronisation.
#pragma once
#include "pluq_basecase.cuh"

namespace pluq {

struct SmallCtx {
  ModP mp;
  int threshold;
  Counts* cnt;      // shared, touched by thread 0 only
  BcShared* sh;
  const uint16_t* invtab;  // inverses mod p when p < 2^16, else nullptr
  int try_generic;         // attempt the generic-profile Crout at internal nodes (depth >= try_depth)
  int try_depth;
};

// OpCounts of the reference recursion on a generic-profile block (see pluq_driver.cu).
PLUQ_HD void generic_counts_dev(int64_t m, int64_t n, int64_t rho, int64_t thr, Counts& c) {
  if (m == 0 || n == 0) return;
  const int64_t rr = (m < n ? m : n) < rho ? (m < n ? m : n) : rho;
  if (m == 1 || n == 1 || (m < n ? m : n) <= thr) {
    for (int64_t t = 0; t < rr; ++t) {
      const long long below = m - 1 - t, right = n - 1 - t;
      if (below > 0) {
        c.inv += 1; c.mul += below; c.red += below;
        if (right > 0) { c.mul += below * right; c.add += below * right; c.red += below * right; }
      }
    }
    return;
  }
  const int64_t kr = m / 2, kc = n / 2;
  int64_t r1 = kr < kc ? kr : kc; r1 = r1 < rho ? r1 : rho;
  generic_counts_dev(kr, kc, rho, thr, c);
  charge_trsm_l(c, r1, n - kc);
  charge_trsm_u(c, m - kr, r1);
  charge_mm(c, kr - r1, n - kc, r1);
  charge_mm(c, m - kr, kc - r1, r1);
  charge_mm(c, m - kr, n - kc, r1);
  int64_t r2 = (kr - r1) < (n - kc) ? (kr - r1) : (n - kc); r2 = r2 < rho - r1 ? r2 : rho - r1;
  generic_counts_dev(kr - r1, n - kc, rho - r1, thr, c);
  int64_t r3 = (m - kr) < (kc - r1) ? (m - kr) : (kc - r1); r3 = r3 < rho - r1 - r2 ? r3 : rho - r1 - r2;
  generic_counts_dev(m - kr, kc - r1, rho - r1 - r2, thr, c);
  const int64_t m4 = m - kr - r3, n4 = n - kc - r2;
  charge_trsm_u(c, r3, r2);
  charge_trsm_l(c, r3, r2);
  charge_trsm_u(c, m4, r2);
  charge_trsm_l(c, r3, n4);
  charge_mm(c, r3, n4, r2);
  charge_mm(c, m4, n4, r2);
  charge_mm(c, m4, n4, r3);
  generic_counts_dev(m4, n4, rho - r1 - r2 - r3, thr, c);
}

__device__ __forceinline__ void cta_ident(int* a, int n) {
  for (int t = threadIdx.x; t < n; t += blockDim.x) a[t] = t;
}

__device__ __forceinline__ bool cta_is_ident(const int* g, int n) {
  bool ok = true;
  for (int t = threadIdx.x; t < n; t += blockDim.x) ok &= (g[t] == t);
  return __syncthreads_and(ok);
}

__device__ __forceinline__ void cta_inverse(const int* g, int* out, int n) {
  for (int t = threadIdx.x; t < n; t += blockDim.x) out[g[t]] = t;
  __syncthreads();
}

// Cycle decomposition of gather vector g (new[x] = old[g[x]]), built by thread 0.
// seq lists each cycle as s, g[s], g[g[s]], ...; lens[c] its length. Returns #cycles.
__device__ __forceinline__ int cta_cycles(const int* g, int n, int* seq, int* lens, int* mark, BcShared* sh) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < n; ++s) mark[s] = 0;
    int pos = 0, nc = 0;
    for (int s = 0; s < n; ++s) {
      if (mark[s] || g[s] == s) continue;
      int cur = s, len = 0;
      do { seq[pos++] = cur; mark[cur] = 1; cur = g[cur]; ++len; } while (cur != s);
      lens[nc++] = len;
    }
    sh->minv = nc;
  }
  __syncthreads();
  int nc = sh->minv;
  __syncthreads();
  return nc;
}

// In-place row gather of view v: new row x = old row g[x] (matrix.py:249-276 semantics).
__device__ void cta_gather_rows(const View v, const int* g, int* scratch, BcShared* sh) {
  if (v.m == 0 || v.n == 0 || cta_is_ident(g, v.m)) return;
  int* seq = scratch; int* lens = seq + v.m; int* mark = lens + v.m;
  int nc = cta_cycles(g, v.m, seq, lens, mark, sh);
  for (int c = threadIdx.x; c < v.n; c += blockDim.x) {
    int pos = 0;
    for (int cy = 0; cy < nc; ++cy) {
      int len = lens[cy];
      uint32_t tmp = v.at(seq[pos], c);
      for (int q = 0; q + 1 < len; ++q) v.at(seq[pos + q], c) = v.at(seq[pos + q + 1], c);
      v.at(seq[pos + len - 1], c) = tmp;
      pos += len;
    }
  }
  __syncthreads();
}

// In-place column gather: new column x = old column g[x].
__device__ void cta_gather_cols(const View v, const int* g, int* scratch, BcShared* sh) {
  if (v.m == 0 || v.n == 0 || cta_is_ident(g, v.n)) return;
  int* seq = scratch; int* lens = seq + v.n; int* mark = lens + v.n;
  int nc = cta_cycles(g, v.n, seq, lens, mark, sh);
  for (int rr = threadIdx.x; rr < v.m; rr += blockDim.x) {
    uint32_t* row = v.row(rr);
    int pos = 0;
    for (int cy = 0; cy < nc; ++cy) {
      int len = lens[cy];
      uint32_t tmp = row[seq[pos]];
      for (int q = 0; q + 1 < len; ++q) row[seq[pos + q]] = row[seq[pos + q + 1]];
      row[seq[pos + len - 1]] = tmp;
      pos += len;
    }
  }
  __syncthreads();
}

// C <- C - A B mod p (kernels.py:38-55), outputs spread over the CTA
// (C column lanes x R row lanes, no integer division in the index math).
__device__ void cta_mm_sub(const View c, const View a, const View b, const ModP mp) {
  const int m = c.m, n = c.n, k = a.n;
  if (m == 0 || n == 0 || k == 0) return;
  const int nt = blockDim.x;
  int C = 1;
  while (C < n && C < nt) C <<= 1;
  const int R = nt / C, tc = threadIdx.x & (C - 1), tr = threadIdx.x / C;
  const bool fast = (uint64_t)k <= mp.kchunk;
  for (int i = tr; i < m; i += R) {
    const uint32_t* ar = a.row(i);
    uint32_t* cr = c.row(i);
    for (int j = tc; j < n; j += C) {
      uint64_t acc = 0;
      if (fast) {
        for (int t = 0; t < k; ++t) acc += (uint64_t)ar[t] * b.at(t, j);
      } else {
        uint64_t cntk = 0;
        for (int t = 0; t < k; ++t) {
          acc += (uint64_t)ar[t] * b.at(t, j);
          if (++cntk == mp.kchunk) { acc = reduce64(acc, mp); cntk = 0; }
        }
      }
      cr[j] = submod(cr[j], reduce64(acc, mp), mp);
    }
  }
  __syncthreads();
}

// B <- L^-1 B, L unit lower (kernels.py:59-83), right-looking over 16-row blocks.
// All 16x16 diagonal blocks are inverted up front in parallel (thread per block
// column); each block solve is then a parallel product X_b = Linv_b B_b followed by
// the rank-16 update of the rows below.  `scr` needs 16*r words.
template <bool fast>
__device__ void cta_trsm_llu_t(const View l, const View b, const ModP mp, uint32_t* scr) {
  const int r = l.m, n = b.n;
  constexpr int BS = 16;
  const int nb = (r + BS - 1) / BS, nt = blockDim.x, tid = threadIdx.x;
  // Linv blocks: scr[blk*256 + i*16 + j]
  for (int t = tid; t < nb * BS; t += nt) {
    const int blk = t / BS, j = t % BS, b0 = blk * BS, bw = min(BS, r - b0);
    uint32_t* X = scr + blk * BS * BS;
    if (j < bw) {
      for (int i = 0; i < j; ++i) X[i * BS + j] = 0u;
      X[j * BS + j] = 1u;
      for (int i = j + 1; i < bw; ++i) {
        uint64_t acc = 0;
        for (int q = j; q < i; ++q) {
          acc += (uint64_t)l.at(b0 + i, b0 + q) * X[q * BS + j];
          if constexpr (!fast) acc = reduce64(acc, mp);
        }
        const uint32_t sv = reduce64(acc, mp);
        X[i * BS + j] = sv ? mp.p - sv : 0u;
      }
    }
  }
  __syncthreads();
  for (int b0 = 0; b0 < r; b0 += BS) {
    const int bw = min(BS, r - b0);
    const uint32_t* X = scr + (b0 / BS) * BS * BS;
    // X_b = Linv_b * B_b : thread per column (owns all bw rows, no hazard)
    for (int col = tid; col < n; col += nt) {
      uint32_t bv[BS];
#pragma unroll
      for (int q = 0; q < BS; ++q) bv[q] = q < bw ? b.at(b0 + q, col) : 0u;
#pragma unroll
      for (int i = 0; i < BS; ++i) {
        if (i >= bw) break;
        uint64_t acc = 0;
#pragma unroll
        for (int q = 0; q <= i; ++q) {
          acc += (uint64_t)X[i * BS + q] * bv[q];
          if constexpr (!fast) acc = reduce64(acc, mp);
        }
        b.at(b0 + i, col) = reduce64(acc, mp);
      }
    }
    __syncthreads();
    const int rest = r - b0 - bw;
    if (rest > 0) {
      for (int idx = tid; idx < rest * n; idx += nt) {
        const int i = b0 + bw + idx / n, c = idx % n;
        const uint32_t* lr = l.row(i) + b0;
        uint64_t acc = 0;
        if constexpr (fast) {
          for (int q = 0; q < bw; ++q) acc += (uint64_t)lr[q] * b.at(b0 + q, c);
        } else {
          for (int q = 0; q < bw; ++q) acc = reduce64(acc + (uint64_t)lr[q] * b.at(b0 + q, c), mp);
        }
        b.at(i, c) = submod(b.at(i, c), reduce64(acc, mp), mp);
      }
      __syncthreads();
    }
  }
}

// B <- B U^-1, U upper with nonzero diagonal (kernels.py:85-120), left-to-right over
// 16-column blocks with all diagonal-block inverses computed up front in parallel.
// `scr` needs 16*r + r words.
template <bool fast>
__device__ void cta_trsm_ru_t(const View b, const View u, uint32_t* scr, const ModP mp, const uint16_t* invtab) {
  const int m = b.m, r = u.m;
  constexpr int BS = 16;
  const int nb = (r + BS - 1) / BS, nt = blockDim.x, tid = threadIdx.x;
  uint32_t* dinv = scr + nb * BS * BS;
  for (int j = tid; j < r; j += nt) dinv[j] = pivot_inverse(u.at(j, j), mp, invtab);
  __syncthreads();
  // Uinv blocks: thread per (block, column j), back substitution within the block
  for (int t = tid; t < nb * BS; t += nt) {
    const int blk = t / BS, j = t % BS, b0 = blk * BS, bw = min(BS, r - b0);
    uint32_t* X = scr + blk * BS * BS;
    if (j < bw) {
      for (int i = j + 1; i < BS; ++i) X[i * BS + j] = 0u;
      X[j * BS + j] = dinv[b0 + j];
      for (int i = j - 1; i >= 0; --i) {
        uint64_t acc = 0;
        for (int q = i + 1; q <= j; ++q) {
          acc += (uint64_t)u.at(b0 + i, b0 + q) * X[q * BS + j];
          if constexpr (!fast) acc = reduce64(acc, mp);
        }
        const uint32_t sv = reduce64(acc, mp);
        X[i * BS + j] = mulmod(sv ? mp.p - sv : 0u, dinv[b0 + i], mp);
      }
    }
  }
  __syncthreads();
  for (int b0 = 0; b0 < r; b0 += BS) {
    const int bw = min(BS, r - b0);
    const uint32_t* X = scr + (b0 / BS) * BS * BS;
    // row block: X_row = B[row, b0:b0+bw] * Uinv_b ; thread per row (owns its bw entries)
    for (int row = tid; row < m; row += nt) {
      uint32_t* br = b.row(row) + b0;
      uint32_t bv[BS];
#pragma unroll
      for (int q = 0; q < BS; ++q) bv[q] = q < bw ? br[q] : 0u;
#pragma unroll
      for (int j = 0; j < BS; ++j) {
        if (j >= bw) break;
        uint64_t acc = 0;
#pragma unroll
        for (int q = 0; q <= j; ++q) {
          acc += (uint64_t)bv[q] * X[q * BS + j];
          if constexpr (!fast) acc = reduce64(acc, mp);
        }
        br[j] = reduce64(acc, mp);
      }
    }
    __syncthreads();
    const int rest = r - b0 - bw;
    if (rest > 0) {
      for (int idx = tid; idx < m * rest; idx += nt) {
        const int rr = idx / rest, jj = b0 + bw + idx % rest;
        const uint32_t* row = b.row(rr) + b0;
        uint64_t acc = 0;
        if constexpr (fast) {
          for (int q = 0; q < bw; ++q) acc += (uint64_t)row[q] * u.at(b0 + q, jj);
        } else {
          for (int q = 0; q < bw; ++q) acc = reduce64(acc + (uint64_t)row[q] * u.at(b0 + q, jj), mp);
        }
        b.at(rr, jj) = submod(b.at(rr, jj), reduce64(acc, mp), mp);
      }
      __syncthreads();
    }
  }
}

__device__ void cta_trsm_llu(const View l, const View b, const ModP mp, uint32_t* scr) {
  if (l.m == 0 || b.n == 0) return;
  if (mp.kchunk >= 16) cta_trsm_llu_t<true>(l, b, mp, scr);
  else cta_trsm_llu_t<false>(l, b, mp, scr);
}
__device__ void cta_trsm_ru(const View b, const View u, uint32_t* scr, const ModP mp, const uint16_t* invtab) {
  if (u.m == 0 || b.m == 0) return;
  if (mp.kchunk >= 16) cta_trsm_ru_t<true>(b, u, scr, mp, invtab);
  else cta_trsm_ru_t<false>(b, u, scr, mp, invtab);
}

__device__ __forceinline__ void cta_copy(const View dst, const View src) {
  for (int idx = threadIdx.x; idx < dst.m * dst.n; idx += blockDim.x) {
    int i = idx / dst.n, j = idx - i * dst.n;
    dst.at(i, j) = src.at(i, j);
  }
  __syncthreads();
}

// Base case in shared memory (fraction-free, CTA-wide); scratch from the stack.
__device__ int base_smem(const View x, int* P, int* Q, int* stk, SmallCtx& c) {
  const int m = x.m, n = x.n, mn = min(m, n);
  BcScratch s;
  s.prow = reinterpret_cast<uint8_t*>(stk);
  s.pcol = s.prow + m;
  int* p = stk + (m + n + 3) / 4 + 1;
  s.rord = p; p += mn;
  s.cord = p; p += mn;
  s.rowat = p; p += m;
  s.colat = p; p += n;
  uint32_t* scale = reinterpret_cast<uint32_t*>(p); p += m;
  uint32_t* bcol = reinterpret_cast<uint32_t*>(p); p += m;
  int* cyc = p;
  BcShared* sh = c.sh;
  auto gather = [&](const int* rowat, const int* colat, int) {
    cta_gather_rows(x, rowat, cyc, sh);
    cta_gather_cols(x, colat, cyc, sh);
  };
  __syncthreads();
  return basecase_ff(x, P, Q, s, scale, bcol, sh, c.mp, c.invtab, c.cnt, gather);
}

// Row-block permutation S and column-block permutation T (recursive.py:77-99).
__device__ __forceinline__ int s_sigma(int x, int r1, int r2, int r3, int r4, int k) {
  int a = r1 + r2, c = r3 + r4, b = k - a;
  if (x >= a && x < k) return x + c;
  if (x >= k && x < k + c) return x - b;
  return x;
}
__device__ __forceinline__ int t_sigma(int x, int r1, int r2, int r3, int r4, int k) {
  if (x < r1) return x;
  if (x < r1 + r2) return x + (k - r1);
  if (x < r1 + r2 + r3) return x - r2;
  if (x < r1 + r2 + r3 + r4) return x + (k + r2 - (r1 + r2 + r3));
  if (x < k + r2 + r4) return x - (r2 + r4);
  return x;
}

template <bool kCheckTrailing>
__device__ int crout_generic(const View x, const ModP mp, const uint16_t* invtab, BcShared* sh);

#ifdef PLUQ_TRACE
#define TR_MARK(i) do { if (threadIdx.x == 0) tr[i] = clock64(); } while (0)
#else
#define TR_MARK(i) do { } while (0)
#endif
__device__ int rec_smem(const View x, int* P, int* Q, int* stk, SmallCtx& c, int depth = 0) {
  const int m = x.m, n = x.n;
#ifdef PLUQ_TRACE
  long long tr[10];
  TR_MARK(0);
#endif
  BcShared* sh = c.sh;
  if (m == 0 || n == 0) {
    cta_ident(P, m); cta_ident(Q, n); __syncthreads();
    return 0;
  }
  if (m == 1 || n == 1 || min(m, n) <= c.threshold) {
#ifdef PLUQ_TRACE
    const int rb = base_smem(x, P, Q, stk, c);
    if (threadIdx.x == 0 && blockIdx.x == 0)
      printf("TRACE d%d base %dx%d r=%d cyc=%lld\n", depth, m, n, rb, clock64() - tr[0]);
    return rb;
#else
    return base_smem(x, P, Q, stk, c);
#endif
  }
  if (c.try_generic && depth >= c.try_depth) {
    // generic-profile shortcut for the whole subtree (exact; see crout_generic)
    uint32_t* bk = reinterpret_cast<uint32_t*>(stk);
    for (int idx = threadIdx.x; idx < m * n; idx += blockDim.x) bk[idx] = x.at(idx / n, idx % n);
    __syncthreads();
    const int rg = crout_generic<true>(x, c.mp, c.invtab, sh);
    if (rg >= 0) {
      cta_ident(P, m); cta_ident(Q, n);
      if (threadIdx.x == 0) generic_counts_dev(m, n, rg, c.threshold, *c.cnt);
      __syncthreads();
#ifdef PLUQ_TRACE
      if (threadIdx.x == 0 && blockIdx.x == 0)
        printf("TRACE d%d generic-ok %dx%d r=%d cyc=%lld\n", depth, m, n, rg, clock64() - tr[0]);
#endif
      return rg;
    }
    for (int idx = threadIdx.x; idx < m * n; idx += blockDim.x) x.at(idx / n, idx % n) = bk[idx];
    __syncthreads();
  }
  TR_MARK(1);
  const int kr = m / 2, kc = n / 2;
  const ModP mp = c.mp;
  const bool t0 = threadIdx.x == 0;

  int* P1 = stk; int* Q1 = P1 + kr; int* top = Q1 + kc;
  const int r1 = rec_smem(x.sub(0, 0, kr, kc), P1, Q1, top, c, depth + 1);
  TR_MARK(2);
  {
    int* g = top; int* scr = g + max(m, n);
    cta_inverse(P1, g, kr);
    cta_gather_rows(x.sub(0, kc, kr, n - kc), g, scr, sh);
    cta_gather_cols(x.sub(kr, 0, m - kr, kc), Q1, scr, sh);
  }
  cta_trsm_llu(x.sub(0, 0, r1, r1), x.sub(0, kc, r1, n - kc), mp, reinterpret_cast<uint32_t*>(top));
  cta_trsm_ru(x.sub(kr, 0, m - kr, r1), x.sub(0, 0, r1, r1), reinterpret_cast<uint32_t*>(top), mp, c.invtab);
  if (t0) {
    charge_trsm_l(*c.cnt, r1, n - kc);
    charge_trsm_u(*c.cnt, m - kr, r1);
    charge_mm(*c.cnt, kr - r1, n - kc, r1);
    charge_mm(*c.cnt, m - kr, kc - r1, r1);
    charge_mm(*c.cnt, m - kr, n - kc, r1);
  }
  cta_mm_sub(x.sub(r1, kc, kr - r1, n - kc), x.sub(r1, 0, kr - r1, r1), x.sub(0, kc, r1, n - kc), mp);
  // G and H share A = E: one pass over the contiguous column range r1..n
  cta_mm_sub(x.sub(kr, r1, m - kr, n - r1), x.sub(kr, 0, m - kr, r1), x.sub(0, r1, r1, n - r1), mp);

  TR_MARK(3);
  int* P2 = top; int* Q2 = P2 + (kr - r1); top = Q2 + (n - kc);
  const int r2 = rec_smem(x.sub(r1, kc, kr - r1, n - kc), P2, Q2, top, c, depth + 1);
  int* P3 = top; int* Q3 = P3 + (m - kr); top = Q3 + (kc - r1);
  const int r3 = rec_smem(x.sub(kr, r1, m - kr, kc - r1), P3, Q3, top, c, depth + 1);
  TR_MARK(4);
  {
    int* ip3 = top; int* ip2 = ip3 + (m - kr); int* scr = ip2 + (kr - r1);
    cta_inverse(P3, ip3, m - kr);
    cta_inverse(P2, ip2, kr - r1);
    cta_gather_rows(x.sub(kr, kc, m - kr, n - kc), ip3, scr, sh);
    cta_gather_cols(x.sub(kr, kc, m - kr, n - kc), Q2, scr, sh);
    cta_gather_rows(x.sub(kr, 0, m - kr, r1), ip3, scr, sh);
    cta_gather_rows(x.sub(r1, 0, kr - r1, r1), ip2, scr, sh);
    cta_gather_cols(x.sub(0, kc, r1, n - kc), Q2, scr, sh);
    cta_gather_cols(x.sub(0, r1, r1, kc - r1), Q3, scr, sh);
  }
  const View u2 = x.sub(r1, kc, r2, r2);
  const View l3 = x.sub(kr, r1, r3, r3);
  const int m4 = m - kr - r3, n4 = n - kc - r2;
  cta_trsm_ru(x.sub(kr, kc, r3, r2), u2, reinterpret_cast<uint32_t*>(top), mp, c.invtab);                      // I
  View J{reinterpret_cast<uint32_t*>(top), r2, r3, r2};
  int* top2 = top + r3 * r2 + 1;
  cta_copy(J, x.sub(kr, kc, r3, r2));
  cta_trsm_llu(l3, J, mp, reinterpret_cast<uint32_t*>(top2));                                               // J (scratch)
  cta_trsm_ru(x.sub(kr + r3, kc, m4, r2), u2, reinterpret_cast<uint32_t*>(top2), mp, c.invtab);                // K
  cta_trsm_llu(l3, x.sub(kr, kc + r2, r3, n4), mp, reinterpret_cast<uint32_t*>(top2));                      // N
  cta_mm_sub(x.sub(kr, kc + r2, r3, n4), J, x.sub(r1, kc + r2, r2, n4), mp);   // O
  cta_mm_sub(x.sub(kr + r3, kc + r2, m4, n4), x.sub(kr + r3, kc, m4, r2), x.sub(r1, kc + r2, r2, n4), mp);
  cta_mm_sub(x.sub(kr + r3, kc + r2, m4, n4), x.sub(kr + r3, r1, m4, r3), x.sub(kr, kc + r2, r3, n4), mp);
  if (t0) {
    charge_trsm_u(*c.cnt, r3, r2);
    charge_trsm_l(*c.cnt, r3, r2);
    charge_trsm_u(*c.cnt, m4, r2);
    charge_trsm_l(*c.cnt, r3, n4);
    charge_mm(*c.cnt, r3, n4, r2);
    charge_mm(*c.cnt, m4, n4, r2);
    charge_mm(*c.cnt, m4, n4, r3);
  }

  TR_MARK(5);
  int* P4 = top; int* Q4 = P4 + m4; top = Q4 + n4;
  const int r4 = rec_smem(x.sub(kr + r3, kc + r2, m4, n4), P4, Q4, top, c, depth + 1);
  TR_MARK(6);
  {
    int* ip4 = top; int* scr = ip4 + m4;
    cta_inverse(P4, ip4, m4);
    cta_gather_rows(x.sub(kr + r3, 0, m4, kc + r2), ip4, scr, sh);
    cta_gather_cols(x.sub(0, kc + r2, kr + r3, n4), Q4, scr, sh);
  }
  {
    int* is = top; int* tg = is + m; int* scr = tg + n;
    for (int t = threadIdx.x; t < m; t += blockDim.x) is[s_sigma(t, r1, r2, r3, r4, kr)] = t;
    for (int t = threadIdx.x; t < n; t += blockDim.x) tg[t] = t_sigma(t, r1, r2, r3, r4, kc);
    __syncthreads();
    cta_gather_rows(x, is, scr, sh);
    cta_gather_cols(x, tg, scr, sh);
  }
  // P = Diag(P1 Diag(I,P2), P3 Diag(I,P4)) S ; Q = T Diag(Diag(I,Q3) Q1, Diag(I,Q4) Q2)
  for (int t = threadIdx.x; t < m; t += blockDim.x) {
    int y;
    if (t < kr) { int z = P1[t]; y = z < r1 ? z : r1 + P2[z - r1]; }
    else { int z = P3[t - kr]; y = kr + (z < r3 ? z : r3 + P4[z - r3]); }
    P[t] = s_sigma(y, r1, r2, r3, r4, kr);
  }
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    int z = t_sigma(t, r1, r2, r3, r4, kc);
    int y;
    if (z < kc) { int w = z < r1 ? z : r1 + Q3[z - r1]; y = Q1[w]; }
    else { int zz = z - kc; int w = zz < r2 ? zz : r2 + Q4[zz - r2]; y = kc + Q2[w]; }
    Q[t] = y;
  }
  __syncthreads();
#ifdef PLUQ_TRACE
  if (threadIdx.x == 0 && blockIdx.x == 0)
    printf("TRACE d%d node %dx%d r=%d,%d,%d,%d attempt=%lld r1=%lld mid=%lld r23=%lld tail=%lld r4=%lld fin=%lld total=%lld\n",
           depth, m, n, r1, r2, r3, r4, tr[1] - tr[0], tr[2] - tr[1], tr[3] - tr[2], tr[4] - tr[3],
           tr[5] - tr[4], tr[6] - tr[5], clock64() - tr[6], clock64() - tr[0]);
#endif
  return r1 + r2 + r3 + r4;
}

// ------------------------------------------------------------------------------------
// Speculative generic-profile path (no pivoting).
//
// If the leading principal minors of orders 1..r are nonzero and the Schur complement
// after r pivots is zero, the reference recursion returns P = Q = I, rank r and the
// unique unpivoted LU factors, for every threshold (tests/test_generic_profile.py pins
// this against the oracle).  crout_generic() runs a Crout LU on the shared-memory
// block and verifies exactly that condition: it returns the rank on success, or -1
// when the block is not generic (then the caller restores the block and runs the
// exact recursion).  Each L/U entry is one dot product with a single delayed
// reduction, two barriers per pivot.
// ------------------------------------------------------------------------------------
template <bool kCheckTrailing = true>
__device__ int crout_generic(const View x, const ModP mp, const uint16_t* invtab, BcShared* sh) {
  const int m = x.m, n = x.n, mn = min(m, n);
  const int tid = threadIdx.x, nt = blockDim.x;
  uint32_t* __restrict__ A = x.a;
  const int ld = (int)x.ld;
  const bool fast = (uint64_t)mn <= mp.kchunk;
  for (int t = 0; t < mn; ++t) {
    if (!kCheckTrailing) {
      // speculative panel mode: settle the pivot first, so a zero pivot leaves row t and
      // column t untouched for the host-side finish (exact Schur complement check)
      if (tid == 0) {
        uint64_t acc = 0;
        const uint32_t* lt = A + t * ld;
        for (int k = 0; k < t; ++k) acc = fast ? acc + (uint64_t)lt[k] * A[k * ld + t]
                                               : reduce64(acc + (uint64_t)lt[k] * A[k * ld + t], mp);
        sh->minv = (int)submod(A[t * ld + t], reduce64(acc, mp), mp);
      }
      __syncthreads();
      const uint32_t pv = (uint32_t)sh->minv;
      __syncthreads();
      if (pv == 0u) return t;
    }
    // U row t: A[t][j] -= sum_{k<t} L[t][k] U[k][j]      (j >= t)
    // L col t numerators: A[i][t] -= sum_{k<t} L[i][k] U[k][t]   (i > t)
    const int nu = n - t, nl = m - t - 1;
    for (int q = tid; q < nu + nl; q += nt) {
      const int i = q < nu ? t : t + 1 + (q - nu);
      const int j = q < nu ? t + q : t;
      uint64_t acc = 0, acc2 = 0;
      const uint32_t* li = A + i * ld;
      const uint32_t* cj = A + j;
      if (fast) {
        int k = 0;
        for (; k + 3 < t; k += 4) {
          acc += (uint64_t)li[k] * cj[k * ld];
          acc2 += (uint64_t)li[k + 1] * cj[(k + 1) * ld];
          acc += (uint64_t)li[k + 2] * cj[(k + 2) * ld];
          acc2 += (uint64_t)li[k + 3] * cj[(k + 3) * ld];
        }
        for (; k < t; ++k) acc += (uint64_t)li[k] * cj[k * ld];
        acc = reduce64(acc, mp) + (uint64_t)reduce64(acc2, mp);
      } else {
        for (int k = 0; k < t; ++k) acc = reduce64(acc + (uint64_t)li[k] * A[k * ld + j], mp);
      }
      A[i * ld + j] = submod(A[i * ld + j], reduce64(acc, mp), mp);
    }
    __syncthreads();
    const uint32_t piv = A[t * ld + t];
    if (piv == 0u && !kCheckTrailing) return t;  // caller verifies the global Schur complement
    if (piv == 0u) {
      // generic only if the whole Schur complement S[t:, t:] is zero (row t is done)
      bool nz = false;
      for (int j = t + tid; j < n; j += nt) nz |= A[t * ld + j] != 0u;
      const int rows = m - t - 1, cols = n - t;
      for (int q = tid; q < rows * cols; q += nt) {
        const int i = t + 1 + q / cols, j = t + q % cols;
        if (j == t) { nz |= A[i * ld + j] != 0u; continue; }  // column t already reduced
        uint64_t acc = 0;
        const uint32_t* li = A + i * ld;
        if (fast) {
          for (int k = 0; k < t; ++k) acc += (uint64_t)li[k] * A[k * ld + j];
        } else {
          for (int k = 0; k < t; ++k) acc = reduce64(acc + (uint64_t)li[k] * A[k * ld + j], mp);
        }
        nz |= submod(A[i * ld + j], reduce64(acc, mp), mp) != 0u;
      }
      if (__syncthreads_or(nz)) return -1;
      for (int q = tid; q < (m - t) * (n - t); q += nt) A[(t + q / (n - t)) * ld + t + q % (n - t)] = 0u;
      __syncthreads();
      return t;
    }
    const uint32_t inv = pivot_inverse(piv, mp, invtab);
    for (int i = t + 1 + tid; i < m; i += nt) A[i * ld + t] = mulmod(A[i * ld + t], inv, mp);
    __syncthreads();
  }
  return mn;
}

// Worst-case stack words used by rec_smem on an m x n node with the given threshold,
// following its allocation pattern: at most 2(m+n) words of live child permutations,
// then either the transient buffers of this level (gather/cycle scratch, S/T vectors,
// the J scratch of at most ceil(m/2) x ceil(n/2)) or a child's own stack, where every
// child block (A1, F, G, R) is at most ceil(m/2) x ceil(n/2).
inline int64_t small_stack_words(int64_t m, int64_t n, int64_t thr) {
  if (m == 0 || n == 0) return 0;
  const int64_t mx = m > n ? m : n, mn = m < n ? m : n;
  if (m == 1 || n == 1 || mn <= thr)  // base_smem: flags, orders, positions, cycles
    return (m + n + 3) / 4 + 1 + 2 * mn + 3 * m + n + 3 * mx + 8;
  const int64_t hm = (m + 1) / 2, hn = (n + 1) / 2;
  int64_t own = 5 * mx + m + n;                  // S/T vectors + cycle scratch
  int64_t jbuf = hm * hn + 1 + 17 * mx + 300;    // J scratch + TRSM block-inverse scratch
  int64_t child = small_stack_words(hm, hn, thr);
  int64_t t = own > jbuf ? own : jbuf;
  t = t > m * n ? t : m * n;  // generic-attempt backup of the node (at the frame base)
  return 2 * (m + n) + (t > child ? t : child) + 8;
}

}  // namespace pluq
