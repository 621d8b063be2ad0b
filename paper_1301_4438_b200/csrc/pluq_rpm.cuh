// Rank-profile fallback for blocks whose rank profile is not generic.
//
// The reference recursion (Algorithm 1, recursive.py:186-256, with the Algorithm 2
// base case iterative.py:23-91) is rank-profile revealing, and its whole output is a
// function of the rank profile matrix R_A (the 0/1 partial permutation with a one at
// every pivot position, SPEC.md "rank profile matrix"):
//
//   (1) P, Q, rank and the charged OpCounts of Alg.1 on A equal those of Alg.1 on R_A;
//   (2) the packed factors of A are the unpivoted LU of A' = P^T A Q^T
//       (A'[t][u] = A[P^-1(t)][Q(u)]), whose leading minors 1..r are nonzero.
//
// tests/test_rpm_fallback.py pins (1) and (2) against the oracle on thousands of random
// non-generic inputs (all thresholds, tiny primes, rank-deficient and sparse blocks).
// So instead of replaying the deep recursion with field arithmetic (hundreds of
// latency-bound barrier phases per 64x64 block), a block is finished in three short
// phases:
//   a) row-order elimination in shared memory -> R_A (pivot of row i = first nonzero
//      of row i once the earlier pivots are eliminated), one barrier per row;
//   b) Alg.1 replayed symbolically on R_A by one warp (index lists only: a partial
//      permutation has no fill, so every TRSM/GEMM of the recursion is the identity
//      on its pattern) -> P, Q, rank, OpCounts;
//   c) fraction-free right-looking LU of A' (gathered straight from global memory),
//      normalised once at the end with all inverses computed in parallel.
// Register-resident versions of a) and c) (16 warps, rows w + 16 t): lazy 64-bit
// accumulators (rpm_rows_lazy / lu_lazy) or, for p < 2^16, reduced 32-bit residues
// (rpm_rows_eager / lu_eager).  Both can resume from a prefix handed over by the 64x64
// generic kernel: when its t-th leading minor is the first zero one, the first t pivots
// are (k, k), R_A = diag(I_t, R_S) for the Schur complement S, and the LU of A' starts
// at step t (the diagonal pivots come first in the quad-recursive order; checked).
#pragma once
#include "pluq_small.cuh"

namespace pluq {

// a) R_A by row-order elimination.  W: m x n block in shared memory (pitch ld), destroyed.
// rp[i] = column of row i's pivot (-1 if none), cp[j] = row of column j's pivot.
// Warp w owns the rows k with k % nw == w, lanes run over columns; fraction-free update
// row_k <- piv * row_k - W[k][j] * row_i keeps the zero pattern exact without inverses.
__device__ int rpm_rows(uint32_t* W, int ld, int m, int n, const ModP mp, int* rp, int* cp) {
  const unsigned FULL = 0xffffffffu;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, w = tid >> 5, nw = nt >> 5;
  for (int t = tid; t < m; t += nt) rp[t] = -1;
  for (int t = tid; t < n; t += nt) cp[t] = -1;
  int r = 0;
  for (int i = 0; i < m && r < n; ++i) {
    __syncthreads();  // row i is final
    const uint32_t* ri = W + i * ld;
    int j = -1;
    for (int c0 = 0; c0 < n; c0 += 32) {
      const int c = c0 + lane;
      const unsigned bb = __ballot_sync(FULL, c < n && ri[c] != 0u);
      if (bb) { j = c0 + __ffs(bb) - 1; break; }
    }
    if (j < 0) continue;  // zero row (uniform: every warp scanned the same row)
    if (tid == 0) { rp[i] = j; cp[j] = i; }
    ++r;
    const uint32_t piv = ri[j];
    const int first = i + 1 + (((w - (i + 1)) % nw) + nw) % nw;
    for (int k = first; k < m; k += nw) {
      uint32_t* rk = W + k * ld;
      const uint32_t f = rk[j];
      if (f == 0u) continue;  // row k untouched: its own scale stays consistent
      __syncwarp();  // every lane has read f before the lane owning column j clears it
      // the WHOLE row is scaled by piv (row i is zero left of j, so those columns only scale)
      for (int c = lane; c < n; c += 32)
        rk[c] = c < j ? mulmod(piv, rk[c], mp) : c == j ? 0u : submod(mulmod(piv, rk[c], mp), mulmod(f, ri[c], mp), mp);
    }
  }
  __syncthreads();
  return r;
}

// b) Symbolic Alg.1 on R_A, executed by one converged warp.
struct SymCtx {
  const int* rp;   // original row -> original column of its one (or -1)
  const int* cp;   // original column -> original row of its one (or -1)
  int* rpos;       // scratch: local index of an original row inside the current base case
  int* cpos;       // scratch: local index of an original column inside the current base case
  int thr;
  Counts cnt;      // lane 0 accumulates
};

// Alg.2 (iterative.py:23-91) on the partial permutation restricted to rows x cols (both
// lists of original indices in local order).  P[local row] = position, Q[position] =
// local column, pivots first then the rest in local order (iterative.py:82-91).  On a
// partial permutation the frontier walk needs no pivot flags: a row (column) at the
// frontier can only be matched with its own single one.
// Base cases of at most 32 x 32: lr/lc live in lane registers, the frontier walk runs on
// all lanes (two independent shuffles per step), and P, Q and the charges come from
// pivot bitmasks (prefix ORs) instead of per-pivot loops.
__device__ int sym_base32(const int* rows, const int* cols, int m, int n, int* P, int* Q, int* stk,
                          SymCtx& s) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  if (lane < m) s.rpos[rows[lane]] = lane;
  if (lane < n) s.cpos[cols[lane]] = lane;
  __syncwarp();
  int lr = -1, lc = -1;
  if (lane < m) {
    const int x = s.rp[rows[lane]];
    if (x >= 0) {
      const int q = s.cpos[x];
      if ((unsigned)q < (unsigned)n && cols[q] == x) lr = q;
    }
  }
  if (lane < n) {
    const int y = s.cp[cols[lane]];
    if (y >= 0) {
      const int q = s.rpos[y];
      if ((unsigned)q < (unsigned)m && rows[q] == y) lc = q;
    }
  }
  int i = 0, j = 0, r = 0, myro = 0, myco = 0;
  while (i < m || j < n) {
    const int a = __shfl_sync(FULL, lc, j & 31);
    const int b = __shfl_sync(FULL, lr, i & 31);
    int pr, pc;
    if (j < n && a >= 0 && a < i) { pr = a; pc = j; ++j; }           // column segment
    else if (i < m && b >= 0 && b < j) { pr = i; pc = b; ++i; }      // row segment
    else if (i < m && j < n && b == j) { pr = i; pc = j; ++i; ++j; } // corner
    else { i = min(i + 1, m); j = min(j + 1, n); continue; }
    if (lane == r) { myro = pr; myco = pc; }
    ++r;
  }
  const bool piv = lane < r;
  const unsigned rbit = piv ? 1u << myro : 0u, cbit = piv ? 1u << myco : 0u;
  // prefix ORs over the pivots that precede this one, and the full masks
  unsigned pre_r = rbit, pre_c = cbit;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned ur = __shfl_up_sync(FULL, pre_r, o), uc = __shfl_up_sync(FULL, pre_c, o);
    if (lane >= o) { pre_r |= ur; pre_c |= uc; }
  }
  const unsigned rmask = __shfl_sync(FULL, pre_r, 31), cmask = __shfl_sync(FULL, pre_c, 31);
  pre_r &= ~rbit; pre_c &= ~cbit;  // exclusive
  unsigned long long cm = 0, ca = 0, ci = 0;
  if (piv) {
    const int below = m - 1 - myro - __popc((unsigned)((unsigned long long)pre_r >> (myro + 1)));
    const int right = n - 1 - myco - __popc((unsigned)((unsigned long long)pre_c >> (myco + 1)));
    if (below > 0) {
      const unsigned long long br = (unsigned long long)below * right;
      ci = 1; cm = below + br; ca = br;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    cm += __shfl_xor_sync(FULL, cm, o);
    ca += __shfl_xor_sync(FULL, ca, o);
    ci += __shfl_xor_sync(FULL, ci, o);
  }
  if (lane == 0) { s.cnt.mul += cm; s.cnt.add += ca; s.cnt.inv += ci; s.cnt.red += cm; }
  int* at = stk;  // at[row] = pivot index of a pivot row
  if (piv) at[myro] = lane;
  __syncwarp();
  if (lane < m) {
    const unsigned below_mask = (1u << lane) - 1u;
    P[lane] = (rmask >> lane) & 1u ? at[lane] : r + lane - __popc(rmask & below_mask);
  }
  if (piv) Q[lane] = myco;
  if (lane < n && !((cmask >> lane) & 1u)) Q[r + lane - __popc(cmask & ((1u << lane) - 1u))] = lane;
  __syncwarp();
  return r;
}

__device__ int sym_base(const int* rows, const int* cols, int m, int n, int* P, int* Q, int* stk,
                        SymCtx& s) {
  if (m <= 32 && n <= 32) return sym_base32(rows, cols, m, n, P, Q, stk, s);
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  for (int a = lane; a < m; a += 32) s.rpos[rows[a]] = a;
  for (int b = lane; b < n; b += 32) s.cpos[cols[b]] = b;
  __syncwarp();
  int* lr = stk; int* lc = lr + m; int* ro = lc + n; int* co = ro + min(m, n);
  for (int a = lane; a < m; a += 32) {
    const int x = s.rp[rows[a]];
    int b = -1;
    if (x >= 0) {
      const int q = s.cpos[x];
      if ((unsigned)q < (unsigned)n && cols[q] == x) b = q;  // stale scratch entries fail the check
    }
    lr[a] = b;
  }
  for (int b = lane; b < n; b += 32) {
    const int y = s.cp[cols[b]];
    int a = -1;
    if (y >= 0) {
      const int q = s.rpos[y];
      if ((unsigned)q < (unsigned)m && rows[q] == y) a = q;
    }
    lc[b] = a;
  }
  __syncwarp();
  int r = 0;
  if (lane == 0) {
    int i = 0, j = 0;
    while (i < m || j < n) {
      int pr = -1, pc = -1;
      if (j < n) {  // column segment above the frontier (iterative.py:40-44)
        const int a = lc[j];
        if (a >= 0 && a < i) { pr = a; pc = j; ++j; }
      }
      if (pr < 0 && i < m) {  // row segment left of the frontier, then the corner (:45-53)
        const int b = lr[i];
        if (b >= 0 && b < j) { pr = i; pc = b; ++i; }
        else if (j < n && b == j) { pr = i; pc = j; ++i; ++j; }
      }
      if (pr < 0) { i = min(i + 1, m); j = min(j + 1, n); continue; }  // (:54-57)
      ro[r] = pr; co[r] = pc; ++r;
    }
  }
  r = __shfl_sync(FULL, r, 0);
  __syncwarp();
  // charges of iterative.py:59-75 per pivot, from the pivots that precede it
  unsigned long long cm = 0, ca = 0, ci = 0;
  for (int k = lane; k < r; k += 32) {
    const int pr = ro[k], pc = co[k];
    int below = m - 1 - pr, right = n - 1 - pc;
    for (int t = 0; t < k; ++t) { below -= ro[t] > pr; right -= co[t] > pc; }
    if (below > 0) {
      const unsigned long long br = (unsigned long long)below * right;
      ci += 1; cm += below + br; ca += br;
    }
  }
  for (int o = 16; o; o >>= 1) {
    cm += __shfl_xor_sync(FULL, cm, o);
    ca += __shfl_xor_sync(FULL, ca, o);
    ci += __shfl_xor_sync(FULL, ci, o);
  }
  if (lane == 0) { s.cnt.mul += cm; s.cnt.add += ca; s.cnt.inv += ci; s.cnt.red += cm; }
  for (int x = lane; x < m; x += 32) {
    int pos = -1, before = 0;
    for (int t = 0; t < r; ++t) { pos = ro[t] == x ? t : pos; before += ro[t] < x; }
    P[x] = pos >= 0 ? pos : r + x - before;
  }
  for (int x = lane; x < n; x += 32) {
    int pos = -1, before = 0;
    for (int t = 0; t < r; ++t) { pos = co[t] == x ? t : pos; before += co[t] < x; }
    Q[pos >= 0 ? pos : r + x - before] = x;
  }
  __syncwarp();
  return r;
}

// Alg.1 (recursive.py:186-256) on the index lists.  With R_A's pattern the updates
// D, E vanish and F, G, H are the untouched sub-patterns, so a node only reorders its
// row/column lists by the children's permutations and composes P, Q exactly like
// rec_smem; the OpCounts charges are the same closed forms.
__device__ int sym_rec(const int* rows, const int* cols, int m, int n, int* P, int* Q, int* stk,
                       SymCtx& s) {
  const int lane = threadIdx.x & 31;
  if (m == 0 || n == 0) {
    for (int a = lane; a < m; a += 32) P[a] = a;
    for (int b = lane; b < n; b += 32) Q[b] = b;
    __syncwarp();
    return 0;
  }
  if (m == 1 || n == 1 || min(m, n) <= s.thr) return sym_base(rows, cols, m, n, P, Q, stk, s);
  const int kr = m / 2, kc = n / 2;
  int* P1 = stk; int* Q1 = P1 + kr; int* top = Q1 + kc;
  const int r1 = sym_rec(rows, cols, kr, kc, P1, Q1, top, s);
  int* rt = top; int* cl = rt + kr; top = cl + kc;  // P1^T-ordered top rows, Q1-ordered left columns
  for (int a = lane; a < kr; a += 32) rt[P1[a]] = rows[a];
  for (int t = lane; t < kc; t += 32) cl[t] = cols[Q1[t]];
  __syncwarp();
  if (lane == 0) {
    charge_trsm_l(s.cnt, r1, n - kc);
    charge_trsm_u(s.cnt, m - kr, r1);
    charge_mm(s.cnt, kr - r1, n - kc, r1);
    charge_mm(s.cnt, m - kr, kc - r1, r1);
    charge_mm(s.cnt, m - kr, n - kc, r1);
  }
  int* P2 = top; int* Q2 = P2 + (kr - r1); top = Q2 + (n - kc);
  const int r2 = sym_rec(rt + r1, cols + kc, kr - r1, n - kc, P2, Q2, top, s);
  int* P3 = top; int* Q3 = P3 + (m - kr); top = Q3 + (kc - r1);
  const int r3 = sym_rec(rows + kr, cl + r1, m - kr, kc - r1, P3, Q3, top, s);
  int* hr = top; int* hc = hr + (m - kr); top = hc + (n - kc);
  for (int a = lane; a < m - kr; a += 32) hr[P3[a]] = rows[kr + a];
  for (int t = lane; t < n - kc; t += 32) hc[t] = cols[kc + Q2[t]];
  __syncwarp();
  const int m4 = m - kr - r3, n4 = n - kc - r2;
  if (lane == 0) {
    charge_trsm_u(s.cnt, r3, r2);
    charge_trsm_l(s.cnt, r3, r2);
    charge_trsm_u(s.cnt, m4, r2);
    charge_trsm_l(s.cnt, r3, n4);
    charge_mm(s.cnt, r3, n4, r2);
    charge_mm(s.cnt, m4, n4, r2);
    charge_mm(s.cnt, m4, n4, r3);
  }
  int* P4 = top; int* Q4 = P4 + m4; top = Q4 + n4;
  const int r4 = sym_rec(hr + r3, hc + r2, m4, n4, P4, Q4, top, s);
  // P = Diag(P1 Diag(I,P2), P3 Diag(I,P4)) S ; Q = T Diag(Diag(I,Q3) Q1, Diag(I,Q4) Q2)
  for (int t = lane; t < m; t += 32) {
    int y;
    if (t < kr) { const int z = P1[t]; y = z < r1 ? z : r1 + P2[z - r1]; }
    else { const int z = P3[t - kr]; y = kr + (z < r3 ? z : r3 + P4[z - r3]); }
    P[t] = s_sigma(y, r1, r2, r3, r4, kr);
  }
  for (int t = lane; t < n; t += 32) {
    const int z = t_sigma(t, r1, r2, r3, r4, kc);
    int y;
    if (z < kc) { const int w = z < r1 ? z : r1 + Q3[z - r1]; y = Q1[w]; }
    else { const int zz = z - kc; const int w = zz < r2 ? zz : r2 + Q4[zz - r2]; y = kc + Q2[w]; }
    Q[t] = y;
  }
  __syncwarp();
  return r1 + r2 + r3 + r4;
}

// Words of the symbolic recursion stack for an m x n block (children need at most half
// the parent's lists, plus the base case's lr/lc/ro/co).
__host__ __device__ inline int64_t sym_stack_words(int64_t m, int64_t n) {
  return 12 * (m + n) + 64;
}

// b') Parallel symbolic replay (16 warps).  The rank profile matrix of every node of
// Algorithm 1 is R_A restricted to the node's rows x columns, so the split of a node
// needs no child result: A1 = top-left quadrant; F = the top rows that are not A1
// pivots (original order, as P1 leaves them) x the right columns; G = the bottom rows x
// the left columns that are not A1 pivots; H = the bottom rows that are not G pivots x
// the right columns that are not F pivots; and each child's rank is the number of ones
// of R_A inside it.  The root and its four children are split top-down (one warp per
// node), the up to 16 grandchildren (or terminal children) are replayed concurrently
// by the sequential sym_rec (one warp each), then P, Q, rank and the charges are
// composed bottom-up exactly as sym_rec does (recursive.py:248-254).
struct SymNode {
  const int* rows;
  const int* cols;
  int m, n;
  int* P;
  int* Q;
  int r, kind;   // kind: 0 = unused, 1 = split, 2 = replayed sequentially
  int cr[4];     // ranks of the four children (split nodes)
  Counts cnt;
};

__host__ __device__ inline int64_t sym_par_words(int64_t m, int64_t n) {
  return 16 * (m + n)                                   // per-warp rpos/cpos
         + (m + n + 8) + 2 * (m + n) + 8                // level-1 lists, P/Q
         + 4 * ((m + n) / 2 + 8) + 4 * (m + n + 8)      // level-2 lists, P/Q
         + 4 * sym_stack_words(m / 2 + 1, n / 2 + 1)    // terminal level-1 nodes
         + 16 * sym_stack_words(m / 4 + 2, n / 4 + 2)   // level-2 nodes
         + 64;
}

__device__ __forceinline__ bool sym_terminal(int m, int n, int thr) {
  return m == 0 || n == 0 || m == 1 || n == 1 || min(m, n) <= thr;
}

// Split node X (one converged warp): children written to ch[0..3]; lists and P/Q
// storage are bump-allocated from *lp / *pq.
__device__ __noinline__ void sym_split(const SymNode& X, SymNode* ch, int*& lp, int*& pq, const int* rp, const int* cp,
                          int* rpos, int* cpos, int thr) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int m = X.m, n = X.n, kr = m / 2, kc = n / 2;
  for (int a = lane; a < m; a += 32) rpos[X.rows[a]] = a;
  for (int b = lane; b < n; b += 32) cpos[X.cols[b]] = b;
  __syncwarp();
  // local column of row a's one inside X (or -1), local row of column b's one
  auto rowone = [&](int a) -> int {
    const int x = rp[X.rows[a]];
    if (x < 0) return -1;
    const int q = cpos[x];
    return ((unsigned)q < (unsigned)n && X.cols[q] == x) ? q : -1;
  };
  auto colone = [&](int b) -> int {
    const int y = cp[X.cols[b]];
    if (y < 0) return -1;
    const int q = rpos[y];
    return ((unsigned)q < (unsigned)m && X.rows[q] == y) ? q : -1;
  };
  // stable warp compaction of the indices [lo, hi) whose predicate holds
  auto compact = [&](int lo, int hi, const int* src, int* dst, auto pred) -> int {
    int cnt = 0;
    for (int base = lo; base < hi; base += 32) {
      const int i = base + lane;
      const bool keep = i < hi && pred(i);
      const unsigned bal = __ballot_sync(FULL, keep);
      if (keep) dst[cnt + __popc(bal & ((1u << lane) - 1u))] = src[i];
      cnt += __popc(bal);
    }
    return cnt;
  };
  int* Frows = lp; lp += kr;
  const int nF = compact(0, kr, X.rows, Frows, [&](int a) { const int q = rowone(a); return !(q >= 0 && q < kc); });
  int* Gcols = lp; lp += kc;
  const int nG = compact(0, kc, X.cols, Gcols, [&](int b) { const int q = colone(b); return !(q >= 0 && q < kr); });
  const int r1 = kr - nF;
  // F pivots: right columns whose one lies in the top rows; G pivots: bottom rows whose
  // one lies in the left columns (neither can be an A1 pivot)
  int* Hrows = lp; lp += m - kr;
  const int nH = compact(kr, m, X.rows, Hrows, [&](int a) { const int q = rowone(a); return !(q >= 0 && q < kc); });
  int* Hcols = lp; lp += n - kc;
  const int nHc = compact(kc, n, X.cols, Hcols, [&](int b) { const int q = colone(b); return !(q >= 0 && q < kr); });
  const int r3 = (m - kr) - nH, r2 = (n - kc) - nHc;
  __syncwarp();
  if (lane == 0) {
    ch[0] = SymNode{X.rows, X.cols, kr, kc, nullptr, nullptr, 0, 0, {0, 0, 0, 0}, {0, 0, 0, 0}};
    ch[1] = SymNode{Frows, X.cols + kc, nF, n - kc, nullptr, nullptr, 0, 0, {0, 0, 0, 0}, {0, 0, 0, 0}};
    ch[2] = SymNode{X.rows + kr, Gcols, m - kr, nG, nullptr, nullptr, 0, 0, {0, 0, 0, 0}, {0, 0, 0, 0}};
    ch[3] = SymNode{Hrows, Hcols, nH, nHc, nullptr, nullptr, 0, 0, {0, 0, 0, 0}, {0, 0, 0, 0}};
    for (int c = 0; c < 4; ++c) {
      ch[c].P = pq; pq += ch[c].m;
      ch[c].Q = pq; pq += ch[c].n;
      ch[c].kind = sym_terminal(ch[c].m, ch[c].n, thr) ? 2 : 1;
    }
    (void)r1; (void)r2; (void)r3;
  }
  __syncwarp();
}

// P, Q, rank and charges of split node X from its four children (sym_rec's tail).
__device__ void sym_compose(SymNode& X, const SymNode* ch) {
  const int lane = threadIdx.x & 31;
  const int m = X.m, n = X.n, kr = m / 2, kc = n / 2;
  const int r1 = ch[0].r, r2 = ch[1].r, r3 = ch[2].r, r4 = ch[3].r;
  const int* P1 = ch[0].P; const int* Q1 = ch[0].Q;
  const int* P2 = ch[1].P; const int* Q2 = ch[1].Q;
  const int* P3 = ch[2].P; const int* Q3 = ch[2].Q;
  const int* P4 = ch[3].P; const int* Q4 = ch[3].Q;
  for (int t = lane; t < m; t += 32) {
    int y;
    if (t < kr) { const int z = P1[t]; y = z < r1 ? z : r1 + P2[z - r1]; }
    else { const int z = P3[t - kr]; y = kr + (z < r3 ? z : r3 + P4[z - r3]); }
    X.P[t] = s_sigma(y, r1, r2, r3, r4, kr);
  }
  for (int t = lane; t < n; t += 32) {
    const int z = t_sigma(t, r1, r2, r3, r4, kc);
    int y;
    if (z < kc) { const int w = z < r1 ? z : r1 + Q3[z - r1]; y = Q1[w]; }
    else { const int zz = z - kc; const int w = zz < r2 ? zz : r2 + Q4[zz - r2]; y = kc + Q2[w]; }
    X.Q[t] = y;
  }
  if (lane == 0) {
    Counts c{0, 0, 0, 0};
    for (int q = 0; q < 4; ++q) {
      c.mul += ch[q].cnt.mul; c.add += ch[q].cnt.add; c.inv += ch[q].cnt.inv; c.red += ch[q].cnt.red;
    }
    charge_trsm_l(c, r1, n - kc);
    charge_trsm_u(c, m - kr, r1);
    charge_mm(c, kr - r1, n - kc, r1);
    charge_mm(c, m - kr, kc - r1, r1);
    charge_mm(c, m - kr, n - kc, r1);
    const int m4 = m - kr - r3, n4 = n - kc - r2;
    charge_trsm_u(c, r3, r2);
    charge_trsm_l(c, r3, r2);
    charge_trsm_u(c, m4, r2);
    charge_trsm_l(c, r3, n4);
    charge_mm(c, r3, n4, r2);
    charge_mm(c, m4, n4, r2);
    charge_mm(c, m4, n4, r3);
    X.cnt = c;
    X.r = r1 + r2 + r3 + r4;
  }
  __syncwarp();
}

// All threads of the CTA (>= 16 warps).  Returns the rank; P, Q, cnt_out as sym_rec.
__device__ __noinline__ int sym_par(const int* rows, const int* cols, int m, int n, int* P, int* Q, int thr, const int* rp,
                       const int* cp, int* scratch, int* stk_seq, Counts* cnt_out) {
  __shared__ SymNode nd[21];  // root, 4 children, 16 grandchildren
  __shared__ int s_rank;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int* rposw = scratch + w * (m + n);
  int* cposw = rposw + m;
  int* sp = scratch + 16 * (m + n);
  int* l1_lists = sp; sp += m + n + 8;
  int* l1_pq = sp; sp += 2 * (m + n) + 8;
  int* l2_lists = sp; sp += 4 * ((m + n) / 2 + 8);
  int* l2_pq = sp; sp += 4 * (m + n + 8);
  const int big = (int)sym_stack_words(m / 2 + 1, n / 2 + 1), small = (int)sym_stack_words(m / 4 + 2, n / 4 + 2);
  int* big_stk = sp; sp += 4 * big;
  int* small_stk = sp;
  if (sym_terminal(m, n, thr)) {  // whole block replayed by one warp
    if (w == 0) {
      SymCtx s{rp, cp, rposw, cposw, thr, {0, 0, 0, 0}};
      const int r = sym_rec(rows, cols, m, n, P, Q, stk_seq, s);
      if (lane == 0) { *cnt_out = s.cnt; s_rank = r; }
    }
    __syncthreads();
    return s_rank;
  }
  if (w == 0) {
    if (lane == 0) nd[0] = SymNode{rows, cols, m, n, P, Q, 0, 1, {0, 0, 0, 0}, {0, 0, 0, 0}};
    __syncwarp();
    int* lp = l1_lists; int* pq = l1_pq;
    sym_split(nd[0], nd + 1, lp, pq, rp, cp, rposw, cposw, thr);
  }
  __syncthreads();
  if (w < 4 && nd[1 + w].kind == 1) {
    int* lp = l2_lists + w * ((m + n) / 2 + 8);
    int* pq = l2_pq + w * (m + n + 8);
    sym_split(nd[1 + w], nd + 5 + 4 * w, lp, pq, rp, cp, rposw, cposw, thr);
  }
  __syncthreads();
  // replay: level-2 node 5 + w (its parent split), or the terminal level-1 node w / 4
  {
    SymNode* X = nullptr;
    int* stk = nullptr;
    if (nd[1 + w / 4].kind == 1) { X = nd + 5 + w; stk = small_stk + w * small; }
    else if ((w & 3) == 0) { X = nd + 1 + w / 4; stk = big_stk + (w / 4) * big; }
    if (X) {
      SymCtx s{rp, cp, rposw, cposw, thr, {0, 0, 0, 0}};
      const int r = sym_rec(X->rows, X->cols, X->m, X->n, X->P, X->Q, stk, s);
      if (lane == 0) { X->r = r; X->cnt = s.cnt; }
    }
  }
  __syncthreads();
  if (w < 4 && nd[1 + w].kind == 1) sym_compose(nd[1 + w], nd + 5 + 4 * w);
  __syncthreads();
  if (w == 0) {
    sym_compose(nd[0], nd + 1);
    if (lane == 0) { *cnt_out = nd[0].cnt; s_rank = nd[0].r; }
  }
  __syncthreads();
  return s_rank;
}

// c) Fraction-free right-looking LU of the generic block W (r pivots on the diagonal),
// then L[k][s] = W[k][s] / W[s][s] and U[s][c] = W[s][c] / prod_{t<s} W[t][t].
// dinv, dpre: r words of scratch each.
__device__ void ff_lu_generic(uint32_t* W, int ld, int m, int n, int r, const ModP mp,
                              const uint16_t* invtab, uint32_t* dinv, uint32_t* dpre) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, w = tid >> 5, nw = nt >> 5;
  for (int s = 0; s < r; ++s) {
    __syncthreads();  // row s is final
    const uint32_t* ps = W + s * ld;
    const uint32_t piv = ps[s];
    if (piv == 0u) __trap();  // impossible for A' = P^T A Q^T (leading minors nonzero)
    const int first = s + 1 + (((w - (s + 1)) % nw) + nw) % nw;
    for (int k = first; k < m; k += nw) {
      uint32_t* rk = W + k * ld;
      const uint32_t f = rk[s];
      // every trailing row is scaled by piv, even when f == 0, so that rows k and s carry
      // the same factor prod_{t<s} W[t][t] at step s (L[k][s] = W[k][s] / W[s][s])
      if (f == 0u) {
        for (int c = s + 1 + lane; c < n; c += 32) rk[c] = mulmod(piv, rk[c], mp);
      } else {
        for (int c = s + 1 + lane; c < n; c += 32)
          rk[c] = submod(mulmod(piv, rk[c], mp), mulmod(f, ps[c], mp), mp);
      }
    }
  }
  __syncthreads();
  for (int s = tid; s < r; s += nt) dinv[s] = pivot_inverse(W[s * ld + s], mp, invtab);
  __syncthreads();
  if (tid == 0) {
    uint32_t acc = 1u;
    for (int s = 0; s < r; ++s) { dpre[s] = acc; acc = mulmod(acc, dinv[s], mp); }
  }
  __syncthreads();
  for (int k = w; k < m; k += nw) {
    uint32_t* rk = W + k * ld;
    const uint32_t us = k < r ? dpre[k] : 0u;
    for (int c = lane; c < n; c += 32) {
      if (c >= k) { if (k < r && us != 1u) rk[c] = mulmod(rk[c], us, mp); }
      else if (c < r) rk[c] = mulmod(rk[c], dinv[c], mp);
    }
  }
  __syncthreads();
}

// ---- register-resident variants of a) and c) (blocks up to 32*NQ columns and NR rows
// per warp: the hot case).  Warp w holds rows k = w + nw*t, lane holds columns
// c = lane + 32*q; the row being eliminated is broadcast through a double-buffered
// shared row and the multipliers through __shfl_sync, so a step costs one barrier and
// touches no shared memory for the rows a warp owns.
template <int NQ>
__device__ __forceinline__ uint32_t lane_pick(const uint32_t (&v)[NQ], int q) {
  uint32_t x = v[0];
#pragma unroll
  for (int u = 1; u < NQ; ++u) x = q == u ? v[u] : x;
  return x;
}

// the owner warp of row k publishes it into rowbuf (32*NQ words)
template <int NQ, int NR>
__device__ __forceinline__ void publish_row(const uint32_t (&a)[NR][NQ], int k, uint32_t* rowbuf) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (k % nw != w) return;
  const int tk = k / nw;
#pragma unroll
  for (int t = 0; t < NR; ++t)
    if (t == tk) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) rowbuf[lane + 32 * q] = a[t][q];
    }
}

template <int NQ, int NR>
__device__ int rpm_rows_reg(const uint32_t* ga, int64_t lda, int m, int n, const ModP mp, int* rp, int* cp,
                            uint32_t* rowbuf) {
  const unsigned FULL = 0xffffffffu;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, w = tid >> 5, nw = nt >> 5;
  uint32_t a[NR][NQ];
#pragma unroll
  for (int t = 0; t < NR; ++t) {
    const int k = w + nw * t;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int c = lane + 32 * q;
      a[t][q] = (k < m && c < n) ? ga[(int64_t)k * lda + c] : 0u;
    }
  }
  for (int t = tid; t < m; t += nt) rp[t] = -1;
  for (int t = tid; t < n; t += nt) cp[t] = -1;
  publish_row<NQ, NR>(a, 0, rowbuf);
  int r = 0;
  for (int i = 0; i < m && r < n; ++i) {
    __syncthreads();  // row i published
    const uint32_t* ri = rowbuf + (i & 1) * (32 * NQ);
    uint32_t rv[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) rv[q] = ri[lane + 32 * q];
    int j = -1;
#pragma unroll
    for (int q = NQ - 1; q >= 0; --q) {
      const unsigned bb = __ballot_sync(FULL, rv[q] != 0u);
      if (bb) j = 32 * q + __ffs(bb) - 1;
    }
    if (j >= 0) {
      if (tid == 0) { rp[i] = j; cp[j] = i; }
      ++r;
      const int jq = j >> 5, jl = j & 31;
      const uint32_t piv = __shfl_sync(FULL, lane_pick<NQ>(rv, jq), jl);
#pragma unroll
      for (int t = 0; t < NR; ++t) {
        const int k = w + nw * t;
        const uint32_t f = __shfl_sync(FULL, lane_pick<NQ>(a[t], jq), jl);
        if (k > i && f != 0u) {  // warp-uniform; rows >= m hold zeros
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            const int c = lane + 32 * q;
            const uint32_t x = mulmod(piv, a[t][q], mp);
            a[t][q] = c < j ? x : c == j ? 0u : submod(x, mulmod(f, rv[q], mp), mp);
          }
        }
      }
    }
    if (i + 1 < m) publish_row<NQ, NR>(a, i + 1, rowbuf + ((i + 1) & 1) * (32 * NQ));
  }
  __syncthreads();
  return r;
}

// c) on registers: A'[k][c] = A[pinv[k]][Q[c]] gathered from global, r pivot steps, the
// packed factors written back to global.  kInv (p < 2^16): multipliers through the
// inverse table, one product per element; else fraction-free with the final
// normalisation of ff_lu_generic.
template <int NQ, int NR, bool kInv>
__device__ void lu_reg(uint32_t* ga, int64_t lda, int m, int n, int r, const int* pinv, const int* Q,
                       const ModP mp, const uint16_t* invtab, uint32_t* rowbuf, uint32_t* diag, uint32_t* dinv,
                       uint32_t* dpre) {
  const unsigned FULL = 0xffffffffu;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, w = tid >> 5, nw = nt >> 5;
  uint32_t a[NR][NQ];
#pragma unroll
  for (int t = 0; t < NR; ++t) {
    const int k = w + nw * t;
    const uint32_t* src = k < m ? ga + (int64_t)pinv[k] * lda : ga;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int c = lane + 32 * q;
      a[t][q] = (k < m && c < n) ? src[Q[c]] : 0u;
    }
  }
  __syncthreads();  // every original row is in registers before any packed row is written
  publish_row<NQ, NR>(a, 0, rowbuf);
  for (int s = 0; s < r; ++s) {
    __syncthreads();
    const uint32_t* rs = rowbuf + (s & 1) * (32 * NQ);
    uint32_t rv[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) rv[q] = rs[lane + 32 * q];
    const int sq = s >> 5, sl = s & 31;
    const uint32_t piv = __shfl_sync(FULL, lane_pick<NQ>(rv, sq), sl);
    if (piv == 0u) __trap();  // impossible for A' (leading minors 1..r nonzero)
    uint32_t inv = 0u;
    if (kInv) inv = invtab[piv];
    else if (tid == 0) diag[s] = piv;
#pragma unroll
    for (int t = 0; t < NR; ++t) {
      const int k = w + nw * t;
      const uint32_t f = __shfl_sync(FULL, lane_pick<NQ>(a[t], sq), sl);
      if (k > s && k < m) {
        if (kInv) {
          if (f != 0u) {
            const uint32_t l = mulmod(f, inv, mp);
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
              const int c = lane + 32 * q;
              if (c > s) a[t][q] = submod(a[t][q], mulmod(l, rv[q], mp), mp);
              else if (c == s) a[t][q] = l;
            }
          }
        } else {
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            const int c = lane + 32 * q;
            if (c > s) a[t][q] = submod(mulmod(piv, a[t][q], mp), mulmod(f, rv[q], mp), mp);
          }
        }
      }
    }
    if (s + 1 < m) publish_row<NQ, NR>(a, s + 1, rowbuf + ((s + 1) & 1) * (32 * NQ));
  }
  if (!kInv) {
    __syncthreads();
    for (int s = tid; s < r; s += nt) dinv[s] = pivot_inverse(diag[s], mp, invtab);
    __syncthreads();
    if (tid == 0) {
      uint32_t acc = 1u;
      for (int s = 0; s < r; ++s) { dpre[s] = acc; acc = mulmod(acc, dinv[s], mp); }
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < NR; ++t) {
      const int k = w + nw * t;
      if (k >= m) continue;
      const uint32_t us = k < r ? dpre[k] : 1u;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int c = lane + 32 * q;
        if (c >= n) continue;
        if (c >= k) { if (k < r) a[t][q] = mulmod(a[t][q], us, mp); }
        else if (c < r) a[t][q] = mulmod(a[t][q], dinv[c], mp);
      }
    }
  }
#pragma unroll
  for (int t = 0; t < NR; ++t) {
    const int k = w + nw * t;
    if (k >= m) continue;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int c = lane + 32 * q;
      if (c < n) ga[(int64_t)k * lda + c] = a[t][q];
    }
  }
}

// ---- lazy-reduction variants of a) and c) for blocks up to 64 x 64 (shape 1, 512
// threads).  Warp w holds rows k = w + 16 t (t < 4), lane holds columns c = lane + 32 q
// (q < 2); every element is a 64-bit accumulator taking ONE IMAD.WIDE per elimination
// step (acc += c_k * w_c) and reduced only when read: the pivot row by its owner warp
// (two values per lane), the pivot column by the lanes 0..3 of each warp after a shuffle
// gather.  A step costs one CTA barrier and ~10 integer instructions per element instead
// of two modular products.  kSmall: p < 2^16, accumulators < 2^38 (two 32-bit Barrett
// steps), inverse table staged in shared memory; else 64 (p-1)^2 + p < 2^64 and Euclid.
template <bool kSmall>
__device__ __forceinline__ uint32_t rl_red(unsigned long long x, const ModP& mp, uint32_t e32) {
  if (kSmall) return reduce32(reduce32((uint32_t)x, mp) + (uint32_t)(x >> 32) * e32, mp);
  return reduce64(x, mp);
}
template <bool kSmall>
__device__ __forceinline__ uint32_t rl_mul(uint32_t a, uint32_t b, const ModP& mp) {
  if (kSmall) return reduce32(a * b, mp);
  return reduce64((unsigned long long)a * b, mp);
}
template <bool kSmall>
__device__ __forceinline__ uint32_t rl_inv(uint32_t d, const ModP& mp, const uint16_t* stab) {
  if (d == 0u) return 0u;
  return kSmall ? (uint32_t)stab[d] : invmod(d, mp);
}
template <int NR, int NQ>
__device__ __forceinline__ unsigned long long rl_sel(const unsigned long long (&a)[NR][NQ], int t, int q) {
  unsigned long long x[NQ];
#pragma unroll
  for (int c = 0; c < NQ; ++c) {
    x[c] = a[0][c];
#pragma unroll
    for (int u = 1; u < NR; ++u) x[c] = t == u ? a[u][c] : x[c];
  }
  unsigned long long y = x[0];
#pragma unroll
  for (int c = 1; c < NQ; ++c) y = q == c ? x[c] : y;
  return y;
}

// Column `col` of this warp's NR rows, reduced by lanes 0..NR-1 (rows k <= lim give 0).
template <bool kSmall, int NR, int NQ>
__device__ __forceinline__ void rl_column(const unsigned long long (&a)[NR][NQ], int col, int lim, int m,
                                          const ModP& mp, uint32_t e32, uint32_t (&cv)[NR]) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int cq = col >> 5, cl = col & 31;
  unsigned long long mine = 0;
#pragma unroll
  for (int t = 0; t < NR; ++t) {
    unsigned long long x = a[t][0];
#pragma unroll
    for (int c = 1; c < NQ; ++c) x = cq == c ? a[t][c] : x;
    const unsigned long long y = __shfl_sync(FULL, x, cl);
    mine = lane == t ? y : mine;
  }
  const uint32_t red = rl_red<kSmall>(mine, mp, e32);
#pragma unroll
  for (int t = 0; t < NR; ++t) {
    const int k = w + 16 * t;
    const uint32_t v = __shfl_sync(FULL, red, t);
    cv[t] = (k > lim && k < m) ? v : 0u;
  }
}

// Stage the inverse table (p < 2^16) into shared memory with cp.async.
__device__ __forceinline__ void rl_stage_table(uint16_t* stab, const uint16_t* tab, uint32_t p) {
  const int words16 = (int)((p + 7) / 8);  // 16-byte chunks covering entries [0, p)
  for (int q = threadIdx.x; q < words16; q += blockDim.x) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(stab + 8 * q);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(tab + 8 * q));
  }
  asm volatile("cp.async.commit_group;\n" ::);
}
__device__ __forceinline__ void rl_wait_table() { asm volatile("cp.async.wait_all;\n" ::); }

// a) R_A by row-order elimination (same outputs as rpm_rows_reg<NQ, NR>), 16 warps:
// warp w holds rows w + 16 t (t < NR), lane holds columns lane + 32 q (q < NQ).
// simg / t0 (optional): the first t0 rows have pivots (k, k) and simg (shared memory,
// pitch 64) holds their unit-lower L and upper U; the elimination then starts at row t0 on
// the Schur complement S = A22 - L21 U12 (R_A = diag(I_t0, R_S)).
template <bool kSmall, int NR, int NQ>
__device__ int rpm_rows_lazy(const uint32_t* ga, int64_t lda, int m, int n, const ModP mp, int* rp, int* cp,
                             const uint16_t* stab, uint32_t* wbuf /* [2][32 NQ] */, int* jbuf /* [2] */,
                             const uint32_t* simg = nullptr, int t0 = 0) {
  const unsigned FULL = 0xffffffffu;
  constexpr int WC = 32 * NQ;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t e32 = kSmall ? (uint32_t)((1ull << 32) % mp.p) : 0u;
  unsigned long long a[NR][NQ];
#pragma unroll
  for (int t = 0; t < NR; ++t) {
    const int k = w + 16 * t;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int c = lane + 32 * q;
      a[t][q] = (k < m && c < n && (!simg || (k >= t0 && c >= t0))) ? ga[(int64_t)k * lda + c] : 0u;
    }
  }
  if (simg && t0 > 0) {  // S = A22 - L21 U12 on this thread's rows >= t0, columns >= t0
    unsigned long long s[NR][NQ];
#pragma unroll
    for (int t = 0; t < NR; ++t)
#pragma unroll
      for (int q = 0; q < NQ; ++q) s[t][q] = 0;
    for (int kk = 0; kk < t0; ++kk) {
      uint32_t u[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int c = lane + 32 * q;
        u[q] = c < n ? simg[kk * 64 + c] : 0u;
      }
#pragma unroll
      for (int t = 0; t < NR; ++t) {
        const int k = w + 16 * t;
        const uint32_t l = k < m ? simg[k * 64 + kk] : 0u;
#pragma unroll
        for (int q = 0; q < NQ; ++q) s[t][q] += (unsigned long long)l * u[q];
      }
    }
#pragma unroll
    for (int t = 0; t < NR; ++t)
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int k = w + 16 * t, c = lane + 32 * q;
        if (k >= t0 && c >= t0 && k < m && c < n) {
          const uint32_t d = rl_red<kSmall>(s[t][q], mp, (uint32_t)((1ull << 32) % mp.p));
          const uint32_t x = (uint32_t)a[t][q];
          a[t][q] = x >= d ? x - d : x + (mp.p - d);
        }
      }
  }
  for (int t = tid; t < m; t += blockDim.x) rp[t] = t < t0 ? t : -1;
  for (int t = tid; t < n; t += blockDim.x) cp[t] = t < t0 ? t : -1;
  if (kSmall) rl_wait_table();
  __syncthreads();  // table staged, rp/cp initialised
  // the owner warp of row i finds its first nonzero column and publishes -row / pivot
  auto publish = [&](int i) {
    if (w != (i & 15)) return;
    const int ti = i >> 4;
    uint32_t u[NQ];
    int j = -1;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      u[q] = rl_red<kSmall>(rl_sel<NR, NQ>(a, ti, q), mp, e32);
      const unsigned b = __ballot_sync(FULL, u[q] != 0u && lane + 32 * q < n);
      if (j < 0 && b) j = 32 * q + __ffs(b) - 1;
    }
    uint32_t* wb = wbuf + (i & 1) * WC;
    if (j >= 0) {
      uint32_t uj = u[0];
#pragma unroll
      for (int q = 1; q < NQ; ++q) uj = (j >> 5) == q ? u[q] : uj;
      const uint32_t d = __shfl_sync(FULL, uj, j & 31);
      const uint32_t iv = rl_inv<kSmall>(d, mp, stab);
#pragma unroll
      for (int q = 0; q < NQ; ++q) wb[lane + 32 * q] = u[q] ? rl_mul<kSmall>(mp.p - u[q], iv, mp) : 0u;
      if (lane == 0) { rp[i] = j; cp[j] = i; }
    }
    if (lane == 0) jbuf[i & 1] = j;
  };
  if (t0 < m) publish(t0);
  int r = t0;
  for (int i = t0; i < m && r < n; ++i) {
    __syncthreads();  // row i published
    const int j = jbuf[i & 1];
    if (j >= 0) {
      ++r;
      uint32_t cv[NR];
      rl_column<kSmall, NR, NQ>(a, j, i, m, mp, e32, cv);
      const uint32_t* wb = wbuf + (i & 1) * WC;
      uint32_t wq[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) wq[q] = wb[lane + 32 * q];
#pragma unroll
      for (int t = 0; t < NR; ++t)
#pragma unroll
        for (int q = 0; q < NQ; ++q) a[t][q] += (unsigned long long)cv[t] * wq[q];
    }
    if (i + 1 < m && r < n) publish(i + 1);
  }
  __syncthreads();
  return r;
}

// c) unpivoted LU of A'[k][c] = A[pinv[k]][Q[c]] (r nonzero leading pivots), packed
// factors written back to ga.  inv_s: r words of shared scratch.
// simg / t0 (optional, P and Q fix 0..t0-1): the first t0 steps are already done in simg
// (pitch 64, unit-lower L and U of A in its own order), so A' starts from its step-t0
// state: U rows and L columns (scale 1) copied, the rest the permuted Schur complement.
template <bool kSmall, int NR, int NQ>
__device__ void lu_lazy(uint32_t* ga, int64_t lda, int m, int n, int r, const int* pinv, const int* Q,
                        const ModP mp, const uint16_t* stab, uint32_t* wbuf /* [2][32 NQ] */, uint32_t* inv_s,
                        const uint32_t* simg = nullptr, int t0 = 0) {
  const unsigned FULL = 0xffffffffu;
  constexpr int WC = 32 * NQ;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t e32 = kSmall ? (uint32_t)((1ull << 32) % mp.p) : 0u;
  unsigned long long a[NR][NQ];
  if (!simg) t0 = 0;
#pragma unroll
  for (int t = 0; t < NR; ++t) {
    const int k = w + 16 * t;
    const uint32_t* src = k < m ? ga + (int64_t)pinv[k] * lda : ga;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int c = lane + 32 * q;
      a[t][q] = (k < m && c < n && k >= t0 && c >= t0) ? src[Q[c]] : 0u;
    }
  }
  if (t0 > 0) {
    unsigned long long s[NR][NQ];
#pragma unroll
    for (int t = 0; t < NR; ++t)
#pragma unroll
      for (int q = 0; q < NQ; ++q) s[t][q] = 0;
    int qc[NQ], pk[NR];
#pragma unroll
    for (int q = 0; q < NQ; ++q) qc[q] = lane + 32 * q < n ? Q[lane + 32 * q] : 0;
#pragma unroll
    for (int t = 0; t < NR; ++t) pk[t] = w + 16 * t < m ? pinv[w + 16 * t] : 0;
    for (int kk = 0; kk < t0; ++kk) {
      uint32_t u[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) u[q] = simg[kk * 64 + qc[q]];
#pragma unroll
      for (int t = 0; t < NR; ++t) {
        const uint32_t l = simg[pk[t] * 64 + kk];
#pragma unroll
        for (int q = 0; q < NQ; ++q) s[t][q] += (unsigned long long)l * u[q];
      }
    }
#pragma unroll
    for (int t = 0; t < NR; ++t)
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int k = w + 16 * t, c = lane + 32 * q;
        if (k >= m || c >= n) continue;
        if (k >= t0 && c >= t0) {
          const uint32_t d = rl_red<kSmall>(s[t][q], mp, e32);
          const uint32_t x = (uint32_t)a[t][q];
          a[t][q] = x >= d ? x - d : x + (mp.p - d);
        } else if (k < t0 && c >= k) {
          a[t][q] = simg[k * 64 + qc[q]];  // U row k (P fixes k)
        } else {
          a[t][q] = simg[pk[t] * 64 + c];  // L column c < t0, final (scale 1 below)
        }
      }
    for (int c = tid; c < t0; c += blockDim.x) inv_s[c] = 1u;
  }
  __syncthreads();  // every original row is in registers before any packed row is written
  auto publish = [&](int s) {
    if (w != (s & 15)) return;
    const int ts = s >> 4;
    uint32_t u[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) u[q] = rl_red<kSmall>(rl_sel<NR, NQ>(a, ts, q), mp, e32);
    uint32_t us = u[0];
#pragma unroll
    for (int q = 1; q < NQ; ++q) us = (s >> 5) == q ? u[q] : us;
    const uint32_t d = __shfl_sync(FULL, us, s & 31);
    if (d == 0u) __trap();  // impossible for A' (leading minors 1..r nonzero)
    const uint32_t iv = rl_inv<kSmall>(d, mp, stab);
    uint32_t* wb = wbuf + (s & 1) * WC;
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      wb[lane + 32 * q] = (lane + 32 * q > s && u[q]) ? rl_mul<kSmall>(mp.p - u[q], iv, mp) : 0u;
    if (lane == 0) inv_s[s] = iv;
  };
  if (t0 < r) publish(t0);
  for (int s = t0; s < r; ++s) {
    __syncthreads();  // pivot row s published
    uint32_t cv[NR];
    rl_column<kSmall, NR, NQ>(a, s, s, m, mp, e32, cv);
    const uint32_t* wb = wbuf + (s & 1) * WC;
    uint32_t wq[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) wq[q] = wb[lane + 32 * q];
#pragma unroll
    for (int t = 0; t < NR; ++t)
#pragma unroll
      for (int q = 0; q < NQ; ++q) a[t][q] += (unsigned long long)cv[t] * wq[q];
    if (s + 1 < r) publish(s + 1);
  }
  __syncthreads();  // inverses of every pivot published
  // U entries are frozen after their row's pivot step, L entries (c < k) hold the Schur
  // value of their column's step (w_c = 0 afterwards), the trailing block is zero.
#pragma unroll
  for (int t = 0; t < NR; ++t) {
    const int k = w + 16 * t;
    if (k >= m) continue;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int c = lane + 32 * q;
      if (c >= n) continue;
      uint32_t v = rl_red<kSmall>(a[t][q], mp, e32);
      if (c < k && c < r) v = rl_mul<kSmall>(v, inv_s[c], mp);
      else if (k >= r && c >= r) v = 0u;
      ga[(int64_t)k * lda + c] = v;
    }
  }
}

// Eager variants of rpm_rows_lazy / lu_lazy for p < 2^16 (inverse table in shared memory):
// every element is kept reduced, a <- (a + c w) mod p with one 32-bit product and one
// Barrett step ((p-1)^2 + p < 2^32).  The per-step chain then has no 64-bit reductions:
// the pivot column reaches every lane of its row with one 32-bit shuffle and the pivot
// row is published straight from registers.
template <int NR, int NQ>
__device__ __forceinline__ uint32_t re_sel(const uint32_t (&a)[NR][NQ], int t, int q) {
  uint32_t x[NQ];
#pragma unroll
  for (int c = 0; c < NQ; ++c) {
    x[c] = a[0][c];
#pragma unroll
    for (int u = 1; u < NR; ++u) x[c] = t == u ? a[u][c] : x[c];
  }
  uint32_t y = x[0];
#pragma unroll
  for (int c = 1; c < NQ; ++c) y = q == c ? x[c] : y;
  return y;
}
// column `col` of this warp's NR rows, on every lane (rows k <= lim give 0)
template <int NR, int NQ>
__device__ __forceinline__ void re_column(const uint32_t (&a)[NR][NQ], int col, int lim, int m, uint32_t (&cv)[NR]) {
  const int w = threadIdx.x >> 5, cq = col >> 5, cl = col & 31;
#pragma unroll
  for (int t = 0; t < NR; ++t) {
    uint32_t x = a[t][0];
#pragma unroll
    for (int c = 1; c < NQ; ++c) x = cq == c ? a[t][c] : x;
    const uint32_t v = __shfl_sync(0xffffffffu, x, cl);
    const int k = w + 16 * t;
    cv[t] = (k > lim && k < m) ? v : 0u;
  }
}
// S = X - L21 U12 for this thread's elements k >= t0, c >= t0 (X already in a, reduced);
// rows of L and columns of U are read through rk / cc (the identity for R_A, P / Q for A')
template <int NR, int NQ>
__device__ __forceinline__ void re_schur(uint32_t (&a)[NR][NQ], const uint32_t* simg, int t0, const int (&rk)[NR],
                                         const int (&cc)[NQ], int m, int n, const ModP& mp) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long s[NR][NQ];
#pragma unroll
  for (int t = 0; t < NR; ++t)
#pragma unroll
    for (int q = 0; q < NQ; ++q) s[t][q] = 0;
  for (int kk = 0; kk < t0; ++kk) {
    uint32_t u[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) u[q] = simg[kk * 64 + cc[q]];
#pragma unroll
    for (int t = 0; t < NR; ++t) {
      const uint32_t l = simg[rk[t] * 64 + kk];
#pragma unroll
      for (int q = 0; q < NQ; ++q) s[t][q] += (unsigned long long)l * u[q];
    }
  }
  const uint32_t e32 = (uint32_t)((1ull << 32) % mp.p);
#pragma unroll
  for (int t = 0; t < NR; ++t)
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int k = w + 16 * t, c = lane + 32 * q;
      if (k >= t0 && c >= t0 && k < m && c < n) {
        const uint32_t d = rl_red<true>(s[t][q], mp, e32);
        a[t][q] = a[t][q] >= d ? a[t][q] - d : a[t][q] + (mp.p - d);
      }
    }
}

template <int NR, int NQ>
__device__ int rpm_rows_eager(const uint32_t* ga, int64_t lda, int m, int n, const ModP mp, int* rp, int* cp,
                              const uint16_t* stab, uint32_t* wbuf /* [2][32 NQ] */, int* jbuf /* [2] */,
                              const uint32_t* simg = nullptr, int t0 = 0) {
  const unsigned FULL = 0xffffffffu;
  constexpr int WC = 32 * NQ;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (!simg) t0 = 0;
  uint32_t a[NR][NQ];
  int rk[NR], cc[NQ];
#pragma unroll
  for (int t = 0; t < NR; ++t) {
    const int k = w + 16 * t;
    rk[t] = k < m ? k : 0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int c = lane + 32 * q;
      cc[q] = c < n ? c : 0;
      a[t][q] = (k < m && c < n && k >= t0 && c >= t0) ? ga[(int64_t)k * lda + c] : 0u;
    }
  }
  if (t0 > 0) re_schur<NR, NQ>(a, simg, t0, rk, cc, m, n, mp);
  for (int t = tid; t < m; t += blockDim.x) rp[t] = t < t0 ? t : -1;
  for (int t = tid; t < n; t += blockDim.x) cp[t] = t < t0 ? t : -1;
  rl_wait_table();
  __syncthreads();  // table staged, rp/cp initialised
  auto publish = [&](int i) {
    if (w != (i & 15)) return;
    const int ti = i >> 4;
    uint32_t u[NQ];
    int j = -1;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      u[q] = re_sel<NR, NQ>(a, ti, q);
      const unsigned b = __ballot_sync(FULL, u[q] != 0u && lane + 32 * q < n);
      if (j < 0 && b) j = 32 * q + __ffs(b) - 1;
    }
    uint32_t* wb = wbuf + (i & 1) * WC;
    if (j >= 0) {
      uint32_t uj = u[0];
#pragma unroll
      for (int q = 1; q < NQ; ++q) uj = (j >> 5) == q ? u[q] : uj;
      const uint32_t iv = stab[__shfl_sync(FULL, uj, j & 31)];
#pragma unroll
      for (int q = 0; q < NQ; ++q) wb[lane + 32 * q] = u[q] ? reduce32((mp.p - u[q]) * iv, mp) : 0u;
      if (lane == 0) { rp[i] = j; cp[j] = i; }
    }
    if (lane == 0) jbuf[i & 1] = j;
  };
  if (t0 < m) publish(t0);
  int r = t0;
  for (int i = t0; i < m && r < n; ++i) {
    __syncthreads();  // row i published
    const int j = jbuf[i & 1];
    if (j >= 0) {
      ++r;
      uint32_t cv[NR];
      re_column<NR, NQ>(a, j, i, m, cv);
      const uint32_t* wb = wbuf + (i & 1) * WC;
      uint32_t wq[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) wq[q] = wb[lane + 32 * q];
#pragma unroll
      for (int t = 0; t < NR; ++t)
        if (w + 16 * t > i)  // warp-uniform: rows <= i are done
#pragma unroll
          for (int q = 0; q < NQ; ++q) a[t][q] = reduce32(a[t][q] + cv[t] * wq[q], mp);
    }
    if (i + 1 < m && r < n) publish(i + 1);
  }
  __syncthreads();
  return r;
}

template <int NR, int NQ>
__device__ void lu_eager(uint32_t* ga, int64_t lda, int m, int n, int r, const int* pinv, const int* Q,
                         const ModP mp, const uint16_t* stab, uint32_t* wbuf /* [2][32 NQ] */, uint32_t* inv_s,
                         const uint32_t* simg = nullptr, int t0 = 0) {
  const unsigned FULL = 0xffffffffu;
  constexpr int WC = 32 * NQ;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (!simg) t0 = 0;
  uint32_t a[NR][NQ];
  int rk[NR], cc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) cc[q] = lane + 32 * q < n ? Q[lane + 32 * q] : 0;
#pragma unroll
  for (int t = 0; t < NR; ++t) {
    const int k = w + 16 * t;
    rk[t] = k < m ? pinv[k] : 0;
    const uint32_t* src = ga + (int64_t)rk[t] * lda;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int c = lane + 32 * q;
      a[t][q] = (k < m && c < n && k >= t0 && c >= t0) ? src[cc[q]] : 0u;
    }
  }
  if (t0 > 0) {
    re_schur<NR, NQ>(a, simg, t0, rk, cc, m, n, mp);
#pragma unroll
    for (int t = 0; t < NR; ++t)
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int k = w + 16 * t, c = lane + 32 * q;
        if (k >= m || c >= n || (k >= t0 && c >= t0)) continue;
        a[t][q] = (k < t0 && c >= k) ? simg[k * 64 + cc[q]]    // U row k (P fixes k)
                                     : simg[rk[t] * 64 + c];   // L column c < t0 (scale 1)
      }
    for (int c = tid; c < t0; c += blockDim.x) inv_s[c] = 1u;
  }
  __syncthreads();  // every original row is in registers before any packed row is written
  auto publish = [&](int s) {
    if (w != (s & 15)) return;
    const int ts = s >> 4;
    uint32_t u[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) u[q] = re_sel<NR, NQ>(a, ts, q);
    uint32_t us = u[0];
#pragma unroll
    for (int q = 1; q < NQ; ++q) us = (s >> 5) == q ? u[q] : us;
    const uint32_t d = __shfl_sync(FULL, us, s & 31);
    if (d == 0u) __trap();  // impossible for A' (leading minors 1..r nonzero)
    const uint32_t iv = stab[d];
    uint32_t* wb = wbuf + (s & 1) * WC;
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      wb[lane + 32 * q] = (lane + 32 * q > s && u[q]) ? reduce32((mp.p - u[q]) * iv, mp) : 0u;
    if (lane == 0) inv_s[s] = iv;
  };
  if (t0 < r) publish(t0);
  for (int s = t0; s < r; ++s) {
    __syncthreads();  // pivot row s published
    uint32_t cv[NR];
    re_column<NR, NQ>(a, s, s, m, cv);
    const uint32_t* wb = wbuf + (s & 1) * WC;
    uint32_t wq[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) wq[q] = wb[lane + 32 * q];
#pragma unroll
    for (int t = 0; t < NR; ++t)
      if (w + 16 * t > s)  // warp-uniform: rows <= s are final
#pragma unroll
        for (int q = 0; q < NQ; ++q) a[t][q] = reduce32(a[t][q] + cv[t] * wq[q], mp);
    if (s + 1 < r) publish(s + 1);
  }
  __syncthreads();  // inverses of every pivot published
#pragma unroll
  for (int t = 0; t < NR; ++t) {
    const int k = w + 16 * t;
    if (k >= m) continue;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int c = lane + 32 * q;
      if (c >= n) continue;
      uint32_t v = a[t][q];
      if (c < k && c < r) v = reduce32(v * inv_s[c], mp);
      else if (k >= r && c >= r) v = 0u;
      ga[(int64_t)k * lda + c] = v;
    }
  }
}

// Shared-memory words of rpm_pluq_block for an m x n block.
__host__ __device__ inline int64_t rpm_smem_words(int64_t m, int64_t n) {
  const int64_t mn = m < n ? m : n;
  return m * n + 6 * (m + n) + 3 * mn + 256 + sym_stack_words(m, n) + 16;
}

}  // namespace pluq
