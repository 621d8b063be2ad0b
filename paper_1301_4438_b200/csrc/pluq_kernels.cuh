// Global-memory kernels used by the host recursion driver and the C ABI.
#pragma once
#include "pluq_small.cuh"
#include "pluq_rpm.cuh"
#include "pluq_diag.cuh"
#include "pluq_diag2.cuh"

namespace pluq {

// Speculative-path predication: kernels launched under a stop flag do nothing once it is set.
__device__ __forceinline__ bool stopped(const int* stop) {
  return stop && *reinterpret_cast<const volatile int*>(stop);
}

// ---------------------------------------------------------------------------------
// Small-node / batched PLUQ: one CTA per block, block staged through shared memory.
// ---------------------------------------------------------------------------------
// Words of one failure-prefix slot (header + the 64 x 65 Crout image of crout_fixed_kernel).
constexpr int kPrefixWords = 4 + 64 * 65;

struct SmallArgs {
  uint32_t* a;          // first block
  int64_t lda;          // row pitch in global memory
  int64_t bstride;      // elements between consecutive blocks of a batch
  int m, n, threshold;
  ModP mp;
  int* p_out;           // batch x m   (P.sigma)
  int* q_out;           // batch x n   (Q.sigma)
  int* r_out;           // batch
  unsigned long long* cnt_out;  // batch x 4 (or 4 if cnt_accumulate)
  int cnt_accumulate;
  const uint16_t* invtab;       // inverse table when p < 2^16 (else nullptr)
  int try_generic;              // attempt the no-pivot generic-profile path first
  int try_depth;                // smallest recursion depth at which small_pluq_kernel attempts it
  const unsigned long long* generic_counts;  // (min(m,n)+1) x 4 charges by rank, or nullptr
  int* generic_flag;            // per block: 1 if the generic path produced the result (or nullptr)
  int* fail_list;               // compacted indices of blocks needing the exact recursion
  int* fail_count;
  int fail_base;                // index offset of this launch's first block in the list
  int lazy = 1;                 // rank-profile kernel: lazy-reduction register phases (shape 1)
  int* done_count = nullptr;    // generic kernel: CTAs finished (streaming fallback consumer)
  int* claim = nullptr;         // rank-profile kernel: next failure-list slot to take (streaming mode)
  int stream_total = 0;         // CTAs of the generic launch (the consumer exits when all are done)
  long long spin_limit = 0;     // consumer: give up waiting after this many cycles (no hang)
  uint32_t* prefix = nullptr;   // per failure slot: [t | 64 x 65 Crout image] of the generic kernel
  int prefix_slots = 0;         // slots available in `prefix`
  int batch_dp = 1;             // 64 x 64 generic kernel: dp2a version (512 <= p < 2^16)
  const int* abort_flag = nullptr;  // batches: set by the asynchronous residue check; every kernel returns at once if set
  int eager = 0;                // rank-profile kernel, p < 2^16: eager (reduced) registers
  int sym_par = 0;              // rank-profile kernel: parallel symbolic replay (scratch in dynamic smem)
  int sym_par_off = 0;          // byte offset of that scratch behind rpm_smem_words (after the table)
};

__device__ void small_pluq_block(const SmallArgs& args, int blk);

// One CTA per block (grid = batch), or - when fail_list is given - a persistent grid
// walking the compacted list of blocks the generic kernel could not finish.
__global__ void small_pluq_kernel(SmallArgs args, const int* fail_list, const int* fail_count) {
  if (args.abort_flag && *reinterpret_cast<const volatile int*>(args.abort_flag)) return;
  if (fail_list) {
    const int cnt = *fail_count;
    for (int q = blockIdx.x; q < cnt; q += gridDim.x) {
      small_pluq_block(args, fail_list[q]);
      __syncthreads();
    }
    return;
  }
  small_pluq_block(args, blockIdx.x);
}

__device__ void small_pluq_block(const SmallArgs& args, int blk) {
  extern __shared__ __align__(16) uint32_t smem_dyn[];
  __shared__ BcShared sh;
  __shared__ Counts cnt;
  const int m = args.m, n = args.n;
  const int lds = n | 1;
  uint32_t* ga = args.a + (int64_t)blk * args.bstride;
  uint32_t* sa = smem_dyn;
  int* stk = reinterpret_cast<int*>(sa + (((int64_t)m * lds + 3) & ~3ll));
  {
    // coalesced staging: warps over rows, lanes over columns, 4 rows in flight per warp
    const int nw = blockDim.x >> 5, w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    for (int i0 = 4 * w; i0 < m; i0 += 4 * nw)
      for (int j = ln; j < n; j += 32) {
        uint32_t v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = i0 + q < m ? ga[(int64_t)(i0 + q) * args.lda + j] : 0u;
#pragma unroll
        for (int q = 0; q < 4; ++q) if (i0 + q < m) sa[(i0 + q) * lds + j] = v[q];
      }
  }
  if (threadIdx.x == 0) { cnt.mul = cnt.add = cnt.inv = cnt.red = 0; }
  __syncthreads();
  SmallCtx c{args.mp, args.threshold, &cnt, &sh, args.invtab, args.try_generic, args.try_depth};
  View x{sa, lds, m, n};
  int* P = stk; int* Q = P + m; int* top = Q + n;
  const int r = rec_smem(x, P, Q, top, c);
  {
    const int nw = blockDim.x >> 5, w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    for (int i = w; i < m; i += nw)
      for (int j = ln; j < n; j += 32) ga[(int64_t)i * args.lda + j] = sa[i * lds + j];
  }
  int* po = args.p_out + (int64_t)blk * m;
  int* qo = args.q_out + (int64_t)blk * n;
  for (int t = threadIdx.x; t < m; t += blockDim.x) po[t] = P[t];
  for (int t = threadIdx.x; t < n; t += blockDim.x) qo[t] = Q[t];
  if (threadIdx.x == 0) {
    args.r_out[blk] = r;
    unsigned long long* co = args.cnt_out + (args.cnt_accumulate ? 0 : 4 * (int64_t)blk);
    if (args.cnt_accumulate) {
      atomicAdd(co + 0, cnt.mul); atomicAdd(co + 1, cnt.add);
      atomicAdd(co + 2, cnt.inv); atomicAdd(co + 3, cnt.red);
    } else {
      co[0] = cnt.mul; co[1] = cnt.add; co[2] = cnt.inv; co[3] = cnt.red;
    }
  }
}

// Exact PLUQ of one block through its rank profile matrix (pluq_rpm.cuh): same outputs
// as small_pluq_block, three short phases instead of the field-arithmetic recursion.
// SHAPE (one code path per instantiation keeps each kernel small): 1 = registers, n <= 64
// and <= 4 rows per warp; 2 = registers, n <= 128 and <= 8 rows per warp; 0 = shared memory.
template <int SHAPE>
__device__ void rpm_pluq_block(const SmallArgs& args, int blk, int slot) {
  extern __shared__ __align__(16) uint32_t smem_dyn[];
  __shared__ Counts s_cnt;
  __shared__ int s_r;
  const int m = args.m, n = args.n, ld = n, mn = min(m, n);
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, w = tid >> 5, nw = nt >> 5;
  uint32_t* ga = args.a + (int64_t)blk * args.bstride;
#ifdef PLUQ_TRACE
  long long tr[6];
#define RPM_MARK(i) do { if (tid == 0) tr[i] = clock64(); } while (0)
#else
#define RPM_MARK(i) do { } while (0)
#endif
  RPM_MARK(0);
  uint32_t* W = smem_dyn;
  int* rp = reinterpret_cast<int*>(W + (int64_t)m * n);
  int* cp = rp + m; int* rpos = cp + n; int* cpos = rpos + m;
  int* P = cpos + n; int* Q = P + m; int* pinv = Q + n; int* rows = pinv + m; int* cols = rows + m;
  uint32_t* dinv = reinterpret_cast<uint32_t*>(cols + n);
  uint32_t* dpre = dinv + mn;
  uint32_t* diag = dpre + mn;
  uint32_t* rowbuf = diag + mn;
  int* stk = reinterpret_cast<int*>(rowbuf + 256);
  constexpr int shape = SHAPE;
  for (int t = tid; t < m; t += nt) rows[t] = t;
  for (int t = tid; t < n; t += nt) cols[t] = t;
  if constexpr (shape == 0) {
    for (int i = w; i < m; i += nw)
      for (int j = lane; j < n; j += 32) W[i * ld + j] = ga[(int64_t)i * args.lda + j];
  }
  __syncthreads();
  RPM_MARK(1);
  int r;
  // shapes 1 and 2: lazy-reduction phases (table staged in shared memory behind the block's
  // words when p < 2^16; else 64-bit accumulators must hold 32 NR products: kchunk check)
  const bool lazy = (shape == 1 || shape == 2) && args.lazy && nt == 512 &&  // rows w + 16 t: 16 warps
                    (args.invtab != nullptr || args.mp.kchunk >= (shape == 1 ? 66u : 130u));
  uint16_t* stab = reinterpret_cast<uint16_t*>(smem_dyn + ((rpm_smem_words(m, n) + 3) & ~3ll));
  if (lazy && args.invtab) rl_stage_table(stab, args.invtab, args.mp.p);
  // prefix from the generic kernel (64 x 64 blocks): the first t0 pivots are (k, k); stage
  // the L/U image (pitch 64) into the unused W region and eliminate only the Schur complement
  int t0 = 0;
  const uint32_t* simg = nullptr;
  if (shape == 1 && lazy && args.invtab && m == 64 && n == 64 && args.prefix && slot >= 0 &&
      slot < args.prefix_slots) {
    const uint32_t* src = args.prefix + (size_t)slot * kPrefixWords;
    t0 = (int)__ldcg(src);
    for (int idx = tid; idx < 64 * 64; idx += nt) W[idx] = __ldcg(src + 4 + (idx >> 6) * 65 + (idx & 63));
    simg = W;
    __syncthreads();
  }
  const bool eager = lazy && args.invtab && args.mp.mu32 && args.eager;
  if constexpr (shape == 1) {
    if (eager) r = rpm_rows_eager<4, 2>(ga, args.lda, m, n, args.mp, rp, cp, stab, rowbuf,
                                        reinterpret_cast<int*>(diag), simg, t0);
    else if (lazy && args.invtab) r = rpm_rows_lazy<true, 4, 2>(ga, args.lda, m, n, args.mp, rp, cp, stab, rowbuf,
                                                           reinterpret_cast<int*>(diag), simg, t0);
    else if (lazy) r = rpm_rows_lazy<false, 4, 2>(ga, args.lda, m, n, args.mp, rp, cp, stab, rowbuf,
                                                  reinterpret_cast<int*>(diag));
    else r = rpm_rows_reg<2, 4>(ga, args.lda, m, n, args.mp, rp, cp, rowbuf);
  } else if constexpr (shape == 2) {
    if (eager) r = rpm_rows_eager<8, 4>(ga, args.lda, m, n, args.mp, rp, cp, stab, rowbuf,
                                        reinterpret_cast<int*>(diag));
    else if (lazy && args.invtab) r = rpm_rows_lazy<true, 8, 4>(ga, args.lda, m, n, args.mp, rp, cp, stab, rowbuf,
                                                           reinterpret_cast<int*>(diag));
    else if (lazy) r = rpm_rows_lazy<false, 8, 4>(ga, args.lda, m, n, args.mp, rp, cp, stab, rowbuf,
                                                  reinterpret_cast<int*>(diag));
    else r = rpm_rows_reg<4, 8>(ga, args.lda, m, n, args.mp, rp, cp, rowbuf);
  }
  else r = rpm_rows(W, ld, m, n, args.mp, rp, cp);
  RPM_MARK(2);
  if (args.sym_par && nw >= 16) {  // parallel replay (scratch behind the table region)
    int* sp = reinterpret_cast<int*>(smem_dyn + ((rpm_smem_words(m, n) + 3) & ~3ll) + (args.sym_par_off >> 2));
    Counts cc;
    const int rs = sym_par(rows, cols, m, n, P, Q, args.threshold, rp, cp, sp, stk, &cc);
    if (tid == 0) { s_cnt = cc; s_r = rs; }
  } else if (tid < 32) {
    SymCtx s{rp, cp, rpos, cpos, args.threshold, {0, 0, 0, 0}};
    const int rs = sym_rec(rows, cols, m, n, P, Q, stk, s);
    if (lane == 0) { s_cnt = s.cnt; s_r = rs; }
  }
  __syncthreads();
  RPM_MARK(3);
  if (s_r != r) __trap();  // the replay must find exactly the pivots of R_A
  for (int t = tid; t < m; t += nt) pinv[P[t]] = t;
  // the prefix pivots (k, k), k < t0, come first in any quad-recursive order; use the
  // prefix for the LU too when P and Q indeed fix them
  bool fixed = true;
  for (int t = tid; t < t0; t += nt) fixed &= P[t] == t && Q[t] == t;
  if (!__syncthreads_and(fixed)) t0 = 0;
  RPM_MARK(4);
  const bool inv = args.invtab != nullptr;
  if constexpr (shape == 1) {
    if (eager) lu_eager<4, 2>(ga, args.lda, m, n, r, pinv, Q, args.mp, stab, rowbuf, dinv, simg, t0);
    else if (lazy && inv) lu_lazy<true, 4, 2>(ga, args.lda, m, n, r, pinv, Q, args.mp, stab, rowbuf, dinv, simg, t0);
    else if (lazy) lu_lazy<false, 4, 2>(ga, args.lda, m, n, r, pinv, Q, args.mp, stab, rowbuf, dinv);
    else if (inv) lu_reg<2, 4, true>(ga, args.lda, m, n, r, pinv, Q, args.mp, args.invtab, rowbuf, diag, dinv, dpre);
    else lu_reg<2, 4, false>(ga, args.lda, m, n, r, pinv, Q, args.mp, args.invtab, rowbuf, diag, dinv, dpre);
  } else if constexpr (shape == 2) {
    if (eager) lu_eager<8, 4>(ga, args.lda, m, n, r, pinv, Q, args.mp, stab, rowbuf, dinv);
    else if (lazy && inv) lu_lazy<true, 8, 4>(ga, args.lda, m, n, r, pinv, Q, args.mp, stab, rowbuf, dinv);
    else if (lazy) lu_lazy<false, 8, 4>(ga, args.lda, m, n, r, pinv, Q, args.mp, stab, rowbuf, dinv);
    else if (inv) lu_reg<4, 8, true>(ga, args.lda, m, n, r, pinv, Q, args.mp, args.invtab, rowbuf, diag, dinv, dpre);
    else lu_reg<4, 8, false>(ga, args.lda, m, n, r, pinv, Q, args.mp, args.invtab, rowbuf, diag, dinv, dpre);
  } else {
    for (int t = w; t < m; t += nw) {  // A'[t][u] = A[P^-1(t)][Q(u)]
      const uint32_t* src = ga + (int64_t)pinv[t] * args.lda;
      for (int u = lane; u < n; u += 32) W[t * ld + u] = src[Q[u]];
    }
    ff_lu_generic(W, ld, m, n, r, args.mp, args.invtab, dinv, dpre);
    for (int i = w; i < m; i += nw)
      for (int j = lane; j < n; j += 32) ga[(int64_t)i * args.lda + j] = W[i * ld + j];
  }
  RPM_MARK(5);
  int* po = args.p_out + (int64_t)blk * m;
  int* qo = args.q_out + (int64_t)blk * n;
  for (int t = tid; t < m; t += nt) po[t] = P[t];
  for (int t = tid; t < n; t += nt) qo[t] = Q[t];
  if (tid == 0) {
    args.r_out[blk] = r;
    unsigned long long* co = args.cnt_out + (args.cnt_accumulate ? 0 : 4 * (int64_t)blk);
    if (args.cnt_accumulate) {
      atomicAdd(co + 0, s_cnt.mul); atomicAdd(co + 1, s_cnt.add);
      atomicAdd(co + 2, s_cnt.inv); atomicAdd(co + 3, s_cnt.red);
    } else {
      co[0] = s_cnt.mul; co[1] = s_cnt.add; co[2] = s_cnt.inv; co[3] = s_cnt.red;
    }
  }
#ifdef PLUQ_TRACE
  if (tid == 0)
    printf("RPM blk %d r=%d shape=%d stage=%lld rows=%lld sym=%lld pinv=%lld lu=%lld total=%lld\n", blk, r, shape,
           tr[1] - tr[0], tr[2] - tr[1], tr[3] - tr[2], tr[4] - tr[3], tr[5] - tr[4], clock64() - tr[0]);
#endif
}

// One CTA per block, or a persistent grid over the failure list of the generic kernel.
// Streaming mode (args.claim): the failure list is consumed while the generic kernel is
// still running.  Slots are taken with a CAS on `claim`; a slot is ready when its entry
// is >= 0 (the list is initialised to -1).  The loop ends when every slot is taken and
// every generic CTA has finished, or after spin_limit cycles without work (a safety
// bound: the kernel launched after the generic one on its stream takes what is left).
__device__ __forceinline__ int rpm_next_slot(const SmallArgs& args, const int* fail_list, const int* fail_count) {
  __shared__ int s_slot;
  if (threadIdx.x == 0) {
    const long long t0 = clock64();
    int got = -1;
    while (true) {
      const int have = *reinterpret_cast<const volatile int*>(fail_count);
      const int q = *reinterpret_cast<volatile int*>(args.claim);
      if (q < have) {
        if (atomicCAS(args.claim, q, q + 1) == q) {
          while (*reinterpret_cast<const volatile int*>(fail_list + q) < 0) __nanosleep(64);
          __threadfence();  // acquire: the slot's prefix image was written before its entry
          got = q;
          break;
        }
        continue;
      }
      if (!args.done_count || *reinterpret_cast<const volatile int*>(args.done_count) >= args.stream_total) {
        // every generic CTA has finished: one last look at the count
        if (q >= *reinterpret_cast<const volatile int*>(fail_count)) break;
        continue;
      }
      if (args.spin_limit && clock64() - t0 > args.spin_limit) break;
      __nanosleep(256);
    }
    s_slot = got;
  }
  __syncthreads();
  const int v = s_slot;
  __syncthreads();
  return v;
}

template <int SHAPE>
__global__ void __launch_bounds__(512, 1) rpm_pluq_kernel(SmallArgs args, const int* fail_list, const int* fail_count) {
  if (args.abort_flag && *reinterpret_cast<const volatile int*>(args.abort_flag)) return;
  if (args.claim) {
    for (int q = rpm_next_slot(args, fail_list, fail_count); q >= 0; q = rpm_next_slot(args, fail_list, fail_count)) {
      rpm_pluq_block<SHAPE>(args, *reinterpret_cast<const volatile int*>(fail_list + q), q);
      __syncthreads();
    }
    return;
  }
  if (fail_list) {
    const int cnt = *fail_count;
    for (int q = blockIdx.x; q < cnt; q += gridDim.x) {
      rpm_pluq_block<SHAPE>(args, fail_list[q], q);
      __syncthreads();
    }
    return;
  }
  rpm_pluq_block<SHAPE>(args, blockIdx.x, -1);
}

// register shape of rpm_pluq_kernel for an m x n block with `threads` per CTA
inline int rpm_shape(int m, int n, int threads) {
  const int nw = threads / 32;
  return (n <= 64 && m <= 4 * nw) ? 1 : (n <= 128 && m <= 8 * nw) ? 2 : 0;
}

inline size_t rpm_smem_bytes(int64_t m, int64_t n, bool table = false) {
  return (size_t)((rpm_smem_words(m, n) + 3) & ~3ll) * 4 + (table ? 65536 * 2 : 0);
}

// Dynamic shared memory of small_pluq_kernel: block (odd pitch) + P/Q + recursion stack.
// Lean generic-profile kernel (no recursion compiled in, so few registers and many
// CTAs per SM): Crout LU + exact genericity check per block.  Successful blocks are
// written back with P = Q = I; failed blocks are left untouched in global memory and
// flagged for small_pluq_kernel, which then runs the exact recursion on them only.
__global__ void crout_fast_kernel(SmallArgs args) {
  if (args.abort_flag && *reinterpret_cast<const volatile int*>(args.abort_flag)) return;
  extern __shared__ __align__(16) uint32_t smem_dyn[];
  __shared__ BcShared sh;
  const int m = args.m, n = args.n;
  const int lds = n | 1;
  uint32_t* ga = args.a + (int64_t)blockIdx.x * args.bstride;
  uint32_t* sa = smem_dyn;
  const int nw = blockDim.x >> 5, w = threadIdx.x >> 5, ln = threadIdx.x & 31;
  for (int i0 = 4 * w; i0 < m; i0 += 4 * nw)
    for (int j = ln; j < n; j += 32) {
      uint32_t v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = i0 + q < m ? ga[(int64_t)(i0 + q) * args.lda + j] : 0u;
#pragma unroll
      for (int q = 0; q < 4; ++q) if (i0 + q < m) sa[(i0 + q) * lds + j] = v[q];
    }
  __syncthreads();
  View x{sa, lds, m, n};
  const int r = crout_generic<true>(x, args.mp, args.invtab, &sh);
  if (threadIdx.x == 0) {
    args.generic_flag[blockIdx.x] = r >= 0;
    if (r < 0 && args.fail_list) atomicExch(args.fail_list + atomicAdd(args.fail_count, 1), args.fail_base + blockIdx.x);
    // streaming batches: the concurrent rank-profile consumer exits once every generic CTA
    // has reported (rpm_next_slot), so failing CTAs count as done too
    if (r < 0 && args.done_count) { __threadfence(); atomicAdd(args.done_count, 1); }
  }
  if (r < 0) return;
  for (int i = w; i < m; i += nw)
    for (int j = ln; j < n; j += 32) ga[(int64_t)i * args.lda + j] = sa[i * lds + j];
  int* po = args.p_out + (int64_t)blockIdx.x * m;
  int* qo = args.q_out + (int64_t)blockIdx.x * n;
  for (int t = threadIdx.x; t < m; t += blockDim.x) po[t] = t;
  for (int t = threadIdx.x; t < n; t += blockDim.x) qo[t] = t;
  if (threadIdx.x == 0) {
    args.r_out[blockIdx.x] = r;
    if (args.done_count) atomicAdd(args.done_count, 1);
    if (args.generic_counts) {
      const unsigned long long* g = args.generic_counts + 4 * r;
      unsigned long long* co = args.cnt_out + (args.cnt_accumulate ? 0 : 4 * (int64_t)blockIdx.x);
      if (args.cnt_accumulate) {
        atomicAdd(co + 0, g[0]); atomicAdd(co + 1, g[1]); atomicAdd(co + 2, g[2]); atomicAdd(co + 3, g[3]);
      } else {
        co[0] = g[0]; co[1] = g[1]; co[2] = g[2]; co[3] = g[3];
      }
    }
  }
}

// Shape-specialised generic-profile kernel (compile-time M x N, M + N - 1 <= NT): Crout
// with ONE barrier per pivot.  Each thread owns one item per step (a U-row entry or an
// L-column numerator).  The L column of step t is published unscaled in a
// double-buffered vector and scaled by its owner during step t+1, while readers apply
// inv(U[t][t]) to that single term themselves; the owner of the pivot publishes its
// inverse before the barrier.  Static shared arrays give immediate-offset LDS.
// kSmall (p < 2^16, with the inverse table): dot-product accumulators stay below 2^38 and
// are reduced with two 32-bit Barrett steps; products of residues fit 32 bits.
// k40 (with kSmall, 512 <= p): the 5-instruction reductions of pluq_diag2.cuh (red40 / mul16).
template <int M, int N, int NT, bool kFast, bool kSmall = false, bool k40 = false>
__global__ void __launch_bounds__(NT) crout_fixed_kernel(SmallArgs args) {
  if (args.abort_flag && *reinterpret_cast<const volatile int*>(args.abort_flag)) return;
  static_assert(M + N - 1 <= NT, "one item per thread per step");
  static_assert(!kSmall || kFast, "the small-prime path is a fast path");
  constexpr int MN = M < N ? M : N;
  constexpr int LD = N | 1;
  __shared__ uint32_t A[M * LD];
  __shared__ uint32_t Ncol[2][M];
  __shared__ uint32_t invs[2];
  __shared__ int zero_at;
  __shared__ BcShared sh;
  const int tid = threadIdx.x;
  const ModP mp = args.mp;
  const uint16_t* tab = args.invtab;
  uint32_t* ga = args.a + (int64_t)blockIdx.x * args.bstride;
  const uint32_t e32 = kSmall ? (uint32_t)((1ull << 32) % mp.p) : 0u;
  const uint32_t P40 = mp.p, NP40 = 0u - mp.p, mu40 = k40 ? (uint32_t)((1ull << 40) / mp.p) : 0u, mu32 = mp.mu32;
  auto mulm = [&](uint32_t a, uint32_t b) -> uint32_t {
    return k40 ? mul16(a, b, P40, NP40, mu32) : kSmall ? reduce32(a * b, mp) : mulmod(a, b, mp);
  };
  auto red = [&](uint64_t x) -> uint32_t {
    return k40      ? red40(x, P40, NP40, mu40)
           : kSmall ? reduce32(reduce32((uint32_t)x, mp) + (uint32_t)(x >> 32) * e32, mp)
                    : reduce64(x, mp);
  };
  {
    // stage the block with cp.async (4-byte copies: the odd row pitch keeps column walks
    // conflict-free) so that all of a thread's loads are in flight at once
    const int w = tid >> 5, ln = tid & 31;
#pragma unroll
    for (int i = w; i < M; i += NT / 32)
#pragma unroll
      for (int j = ln; j < N; j += 32) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(A + i * LD + j);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(ga + (int64_t)i * args.lda + j));
      }
    asm volatile("cp.async.commit_group;\ncp.async.wait_all;\n" ::);
  }
  if (tid == 0) zero_at = -1;
  __syncthreads();
  int own_i = -1;          // L item row owned at the previous step
  uint32_t own_num = 0;    // its unscaled numerator
  uint32_t inv_prev = 0;
  int t = 0;
  for (; t < MN; ++t) {
    const int nu = N - t;
    const bool is_u = tid < nu;
    const bool is_l = !is_u && tid - nu < M - t - 1;
    const int row = is_u ? t : t + 1 + (tid - nu);
    const int col = is_u ? t + tid : t;
    // scale the L entry of the previous step (nobody reads A[.][t-1] during this step)
    if (own_i >= 0) A[own_i * LD + t - 1] = mulm(own_num, inv_prev);
    own_i = -1;
    if (is_u || is_l) {
      uint64_t acc = 0, acc2 = 0;
      const uint32_t* ri = A + row * LD;
      const uint32_t* cj = A + col;
      const int kend = t - 1;  // terms k < t-1 read final values; k = t-1 is the deferred one
      int kk = 0;
      if (kFast) {
#pragma unroll 4
        for (; kk + 1 < kend; kk += 2) {
          acc += (uint64_t)ri[kk] * cj[kk * LD];
          acc2 += (uint64_t)ri[kk + 1] * cj[(kk + 1) * LD];
        }
        if (kk < kend) acc += (uint64_t)ri[kk] * cj[kk * LD];  // at most one term left
        acc += acc2;  // kFast: <= MN products of (p-1)^2 plus one more term fit in 64 bits
      } else {
        for (; kk < kend; ++kk) acc = reduce64(acc + (uint64_t)ri[kk] * cj[kk * LD], mp);
      }
      if (t > 0) {
        const uint32_t lt = mulm(Ncol[(t - 1) & 1][row], inv_prev);  // L[row][t-1]
        acc += (uint64_t)lt * cj[(t - 1) * LD];
      }
      const uint32_t v = submod(A[row * LD + col], red(acc), mp);
      if (is_u) {
        A[row * LD + col] = v;
        if (col == t) {
          if (v == 0u) zero_at = t;
          else invs[t & 1] = (kSmall || tab) ? (uint32_t)tab[v] : invmod(v, mp);
        }
      } else {
        Ncol[t & 1][row] = v;
        own_i = row;
        own_num = v;
      }
    }
    __syncthreads();
    if (zero_at >= 0) break;
    inv_prev = invs[t & 1];
  }
  int r = MN;
  if (zero_at >= 0) {
    // zero pivot at t: column t's Schur values are the unscaled numerators; the
    // previous column's owners already wrote their scaled entries in this step
    for (int i = t + 1 + tid; i < M; i += NT) A[i * LD + t] = Ncol[t & 1][i];
    __syncthreads();
    bool nz = false;
    for (int j = t + tid; j < N; j += NT) nz |= A[t * LD + j] != 0u;
    const int rows = M - t - 1, cols = N - t;
    for (int q = tid; q < rows * cols; q += NT) {
      const int i = t + 1 + q / cols, j = t + q % cols;
      if (j == t) { nz |= A[i * LD + j] != 0u; continue; }
      uint64_t acc = 0;
      for (int kk = 0; kk < t; ++kk) {
        acc += (uint64_t)A[i * LD + kk] * A[kk * LD + j];
        if (!kFast) acc = reduce64(acc, mp);
      }
      nz |= submod(A[i * LD + j], reduce64(acc, mp), mp) != 0u;
    }
    if (__syncthreads_or(nz)) {
      // not generic: the first t pivots are (k, k) and their factors are final in A; hand
      // them to the rank-profile kernel (R_A = diag(I_t, R_S), S the Schur complement)
      __shared__ int s_slot;
      if (tid == 0) s_slot = args.fail_list ? atomicAdd(args.fail_count, 1) : -1;
      __syncthreads();
      const int slot = s_slot;
      if (M == 64 && N == 64 && LD == 65 && args.prefix && slot >= 0 && slot < args.prefix_slots) {
        uint32_t* dst = args.prefix + (size_t)slot * kPrefixWords;
        for (int idx = tid; idx < M * LD; idx += NT) dst[4 + idx] = A[idx];
        if (tid == 0) dst[0] = (uint32_t)t;
        __threadfence();
      }
      __syncthreads();
      if (tid == 0) {
        args.generic_flag[blockIdx.x] = 0;
        if (slot >= 0) atomicExch(args.fail_list + slot, args.fail_base + blockIdx.x);  // a consumer may be waiting
        if (args.done_count) { __threadfence(); atomicAdd(args.done_count, 1); }
      }
      return;
    }
    for (int q = tid; q < (M - t) * (N - t); q += NT) A[(t + q / (N - t)) * LD + t + q % (N - t)] = 0u;
    r = t;
  } else if (own_i >= 0) {
    A[own_i * LD + MN - 1] = mulm(own_num, inv_prev);  // last L column
  }
  __syncthreads();
  {
    const int w = tid >> 5, ln = tid & 31;
    for (int i = w; i < M; i += NT / 32)
      for (int j = ln; j < N; j += 32) ga[(int64_t)i * args.lda + j] = A[i * LD + j];
  }
  int* po = args.p_out + (int64_t)blockIdx.x * M;
  int* qo = args.q_out + (int64_t)blockIdx.x * N;
  for (int q = tid; q < M; q += NT) po[q] = q;
  for (int q = tid; q < N; q += NT) qo[q] = q;
  if (tid == 0) {
    args.generic_flag[blockIdx.x] = 1;
    args.r_out[blockIdx.x] = r;
    if (args.done_count) atomicAdd(args.done_count, 1);
    if (args.generic_counts) {
      const unsigned long long* g = args.generic_counts + 4 * r;
      unsigned long long* co = args.cnt_out + (args.cnt_accumulate ? 0 : 4 * (int64_t)blockIdx.x);
      if (args.cnt_accumulate) {
        atomicAdd(co + 0, g[0]); atomicAdd(co + 1, g[1]); atomicAdd(co + 2, g[2]); atomicAdd(co + 3, g[3]);
      } else {
        co[0] = g[0]; co[1] = g[1]; co[2] = g[2]; co[3] = g[3];
      }
    }
  }
}

// 64 x 64 generic-profile batch kernel for 512 <= p < 2^16, dp2a version of crout_fixed_kernel
// (same schedule: one barrier per pivot, one item per thread per step, L column published
// unscaled and scaled by its owner one step later).  Storage: the block as uint16 (row pitch
// 66: rows are the A operand of the dot products, two consecutive k per 32-bit load) and the
// finished U rows a second time as byte-packed pairs Up[k / 2][j] = [lo(U[2k'][j]),
// lo(U[2k'+1][j]), hi(U[2k'][j]), hi(U[2k'+1][j])], the B operand of IDP.2A: per TWO terms one
// LDS of each operand and two IDP.2A (low and high byte planes, 32-bit accumulators:
// 64 terms x 65535 x 255 < 2^31) instead of four LDS and two IMAD.WIDE (IDP 2.0 vs IMAD.WIDE
// 5.1 cycles per warp instruction, tools/micro/imad_bench.cu).
template <int NT>
__global__ void __launch_bounds__(NT) crout_dp_kernel(SmallArgs args) {
  if (args.abort_flag && *reinterpret_cast<const volatile int*>(args.abort_flag)) return;
  constexpr int M = 64, N = 64, MN = 64, LD = 66, LDI = 65;
  static_assert(M + N - 1 <= NT, "one item per thread per step");
  __shared__ __align__(16) uint16_t A[M * LD];
  __shared__ uint32_t Up[(MN / 2) * N];
  __shared__ uint32_t Ncol[2][M];
  __shared__ uint32_t invs[2];
  __shared__ int zero_at;
  const int tid = threadIdx.x;
  const ModP mp = args.mp;
  const uint16_t* tab = args.invtab;
  uint32_t* ga = args.a + (int64_t)blockIdx.x * args.bstride;
  const uint32_t P = mp.p, NP = 0u - mp.p, mu40 = (uint32_t)((1ull << 40) / mp.p), mu32 = mp.mu32;
  {
    const int w = tid >> 5, ln = tid & 31;
#pragma unroll 4
    for (int i = w; i < M; i += NT / 32) {
      const uint32_t v0 = ga[(int64_t)i * args.lda + ln], v1 = ga[(int64_t)i * args.lda + 32 + ln];
      A[i * LD + ln] = (uint16_t)v0;
      A[i * LD + 32 + ln] = (uint16_t)v1;
    }
  }
  if (tid == 0) zero_at = -1;
  __syncthreads();
  int own_i = -1;          // L item row owned at the previous step
  uint32_t own_num = 0;    // its unscaled numerator
  uint32_t inv_prev = 0;
  int t = 0;
  for (; t < MN; ++t) {
    const int nu = N - t;
    const bool is_u = tid < nu;
    const bool is_l = !is_u && tid - nu < M - t - 1;
    const int row = is_u ? t : t + 1 + (tid - nu);
    const int col = is_u ? t + tid : t;
    // scale the L entry of the previous step (nobody reads A[.][t-1] during this step)
    if (own_i >= 0) A[own_i * LD + t - 1] = (uint16_t)mul16(own_num, inv_prev, P, NP, mu32);
    own_i = -1;
    if (is_u || is_l) {
      uint32_t alo = 0, ahi = 0, alo2 = 0, ahi2 = 0;
      const uint32_t* ri = reinterpret_cast<const uint32_t*>(A + row * LD);  // pairs L[row][2k'], L[row][2k'+1]
      const uint32_t* cj = Up + col;
      const int kend = t - 1;        // terms k < t-1 read final values; k = t-1 is the deferred one
      const int pend = kend >> 1;    // whole pairs
      int kp = 0;
#pragma unroll 4
      for (; kp + 1 < pend; kp += 2) {
        const uint32_t a0 = ri[kp], b0 = cj[kp * N], a1 = ri[kp + 1], b1 = cj[(kp + 1) * N];
        alo = __dp2a_lo(a0, b0, alo);
        ahi = __dp2a_hi(a0, b0, ahi);
        alo2 = __dp2a_lo(a1, b1, alo2);
        ahi2 = __dp2a_hi(a1, b1, ahi2);
      }
      if (kp < pend) {
        const uint32_t a0 = ri[kp], b0 = cj[kp * N];
        alo = __dp2a_lo(a0, b0, alo);
        ahi = __dp2a_hi(a0, b0, ahi);
      }
      unsigned long long acc = (unsigned long long)(alo + alo2) + ((unsigned long long)(ahi + ahi2) << 8);
      if (kend > 0 && (kend & 1)) acc += (uint32_t)A[row * LD + kend - 1] * (uint32_t)A[(kend - 1) * LD + col];  // odd term
      if (t > 0) {
        const uint32_t lt = mul16(Ncol[(t - 1) & 1][row], inv_prev, P, NP, mu32);  // L[row][t-1]
        acc += (unsigned long long)(lt * (uint32_t)A[(t - 1) * LD + col]);
      }
      const uint32_t v = submod((uint32_t)A[row * LD + col], red40(acc, P, NP, mu40), mp);
      if (is_u) {
        A[row * LD + col] = (uint16_t)v;
        uint8_t* ub = reinterpret_cast<uint8_t*>(Up + (t >> 1) * N + col);
        ub[t & 1] = (uint8_t)(v & 255u);
        ub[2 + (t & 1)] = (uint8_t)(v >> 8);
        if (col == t) {
          if (v == 0u) zero_at = t;
          else invs[t & 1] = (uint32_t)tab[v];
        }
      } else {
        Ncol[t & 1][row] = v;
        own_i = row;
        own_num = v;
      }
    }
    __syncthreads();
    if (zero_at >= 0) break;
    inv_prev = invs[t & 1];
  }
  int r = MN;
  if (zero_at >= 0) {
    // zero pivot at t: column t's Schur values are the unscaled numerators; the
    // previous column's owners already wrote their scaled entries in this step
    for (int i = t + 1 + tid; i < M; i += NT) A[i * LD + t] = (uint16_t)Ncol[t & 1][i];
    __syncthreads();
    bool nz = false;
    for (int j = t + tid; j < N; j += NT) nz |= A[t * LD + j] != 0;
    const int rows = M - t - 1, cols = N - t;
    for (int q = tid; q < rows * cols; q += NT) {
      const int i = t + 1 + q / cols, j = t + q % cols;
      if (j == t) { nz |= A[i * LD + j] != 0; continue; }
      unsigned long long acc = 0;
      for (int kk = 0; kk < t; ++kk) acc += (uint32_t)A[i * LD + kk] * (uint32_t)A[kk * LD + j];
      nz |= submod((uint32_t)A[i * LD + j], reduce64(acc, mp), mp) != 0u;
    }
    if (__syncthreads_or(nz)) {
      // not generic: the first t pivots are (k, k) and their factors are final in A; hand
      // them to the rank-profile kernel (R_A = diag(I_t, R_S), S the Schur complement)
      __shared__ int s_slot;
      if (tid == 0) s_slot = args.fail_list ? atomicAdd(args.fail_count, 1) : -1;
      __syncthreads();
      const int slot = s_slot;
      if (args.prefix && slot >= 0 && slot < args.prefix_slots) {
        uint32_t* dst = args.prefix + (size_t)slot * kPrefixWords;
        for (int idx = tid; idx < M * N; idx += NT) dst[4 + (idx >> 6) * LDI + (idx & 63)] = A[(idx >> 6) * LD + (idx & 63)];
        if (tid == 0) dst[0] = (uint32_t)t;
        __threadfence();
      }
      __syncthreads();
      if (tid == 0) {
        args.generic_flag[blockIdx.x] = 0;
        if (slot >= 0) atomicExch(args.fail_list + slot, args.fail_base + blockIdx.x);  // a consumer may be waiting
        if (args.done_count) { __threadfence(); atomicAdd(args.done_count, 1); }
      }
      return;
    }
    for (int q = tid; q < (M - t) * (N - t); q += NT) A[(t + q / (N - t)) * LD + t + q % (N - t)] = 0;
    r = t;
  } else if (own_i >= 0) {
    A[own_i * LD + MN - 1] = (uint16_t)mul16(own_num, inv_prev, P, NP, mu32);  // last L column
  }
  __syncthreads();
  {
    const int w = tid >> 5, ln = tid & 31;
    for (int i = w; i < M; i += NT / 32)
      for (int j = ln; j < N; j += 32) ga[(int64_t)i * args.lda + j] = A[i * LD + j];
  }
  int* po = args.p_out + (int64_t)blockIdx.x * M;
  int* qo = args.q_out + (int64_t)blockIdx.x * N;
  for (int q = tid; q < M; q += NT) po[q] = q;
  for (int q = tid; q < N; q += NT) qo[q] = q;
  if (tid == 0) {
    args.generic_flag[blockIdx.x] = 1;
    args.r_out[blockIdx.x] = r;
    if (args.done_count) atomicAdd(args.done_count, 1);
    if (args.generic_counts) {
      const unsigned long long* g = args.generic_counts + 4 * r;
      unsigned long long* co = args.cnt_out + (args.cnt_accumulate ? 0 : 4 * (int64_t)blockIdx.x);
      if (args.cnt_accumulate) {
        atomicAdd(co + 0, g[0]); atomicAdd(co + 1, g[1]); atomicAdd(co + 2, g[2]); atomicAdd(co + 3, g[3]);
      } else {
        co[0] = g[0]; co[1] = g[1]; co[2] = g[2]; co[3] = g[3];
      }
    }
  }
}

// Launch the generic-profile kernel for a batch: the specialised 64x64 instance when it
// applies, otherwise the runtime-shape kernel.
inline bool launch_crout_fixed(const SmallArgs& a, int64_t batch, cudaStream_t st) {
  if (a.m == 64 && a.n == 64) {
    if (a.mp.mu32 != 0 && a.invtab && a.mp.p >= 512 && a.batch_dp) crout_dp_kernel<128><<<(unsigned)batch, 128, 0, st>>>(a);
    else if (a.mp.mu32 != 0 && a.invtab && a.mp.p >= 512) crout_fixed_kernel<64, 64, 128, true, true, true><<<(unsigned)batch, 128, 0, st>>>(a);
    else if (a.mp.mu32 != 0 && a.invtab) crout_fixed_kernel<64, 64, 128, true, true><<<(unsigned)batch, 128, 0, st>>>(a);
    else if (a.mp.kchunk >= 66) crout_fixed_kernel<64, 64, 128, true><<<(unsigned)batch, 128, 0, st>>>(a);
    else crout_fixed_kernel<64, 64, 128, false><<<(unsigned)batch, 128, 0, st>>>(a);
    return true;
  }
  return false;
}

inline size_t crout_smem_bytes(int64_t m, int64_t n) { return (size_t)(m * (n | 1) + 4) * 4; }

inline size_t small_smem_bytes(int64_t m, int64_t n, int64_t thr) {
  int64_t lds = n | 1;
  return (size_t)((((m * lds) + 3) & ~3ll) + m + n + small_stack_words(m, n, thr) + 64) * 4;
}

// ---------------------------------------------------------------------------------
// Base case on a block too large for shared memory (one CTA, data in global memory).
// ---------------------------------------------------------------------------------
struct BaseArgs {
  View x;
  ModP mp;
  BcScratch s;
  uint32_t* tmp;        // m*n staging for the final gathers
  int* res;             // [m P.sigma | n Q.sigma | rank]
  unsigned long long* cnt_out;  // 4, accumulated
};

__global__ void __launch_bounds__(1024) basecase_global_kernel(BaseArgs args) {
  __shared__ BcShared sh;
  __shared__ Counts cnt;
  if (threadIdx.x == 0) { cnt.mul = cnt.add = cnt.inv = cnt.red = 0; }
  __syncthreads();
  const View x = args.x;
  const int m = x.m, n = x.n;
  uint32_t* tmp = args.tmp;
  auto gather = [&](const int* rowat, const int* colat, int) {
    if (!cta_is_ident(rowat, m)) {
      for (int64_t idx = threadIdx.x; idx < (int64_t)m * n; idx += blockDim.x) {
        int i = (int)(idx / n), j = (int)(idx - (int64_t)i * n);
        tmp[idx] = x.at(rowat[i], j);
      }
      __syncthreads();
      for (int64_t idx = threadIdx.x; idx < (int64_t)m * n; idx += blockDim.x) {
        int i = (int)(idx / n), j = (int)(idx - (int64_t)i * n);
        x.at(i, j) = tmp[idx];
      }
      __syncthreads();
    }
    if (!cta_is_ident(colat, n)) {
      for (int64_t idx = threadIdx.x; idx < (int64_t)m * n; idx += blockDim.x) {
        int i = (int)(idx / n), j = (int)(idx - (int64_t)i * n);
        tmp[idx] = x.at(i, colat[j]);
      }
      __syncthreads();
      for (int64_t idx = threadIdx.x; idx < (int64_t)m * n; idx += blockDim.x) {
        int i = (int)(idx / n), j = (int)(idx - (int64_t)i * n);
        x.at(i, j) = tmp[idx];
      }
      __syncthreads();
    }
  };
  int* P = args.res;
  int* Q = args.res + m;
  int r = basecase_cta(x, P, Q, args.s, &sh, args.mp, &cnt, gather);
  if (threadIdx.x == 0) {
    args.res[m + n] = r;
    atomicAdd(args.cnt_out + 0, cnt.mul); atomicAdd(args.cnt_out + 1, cnt.add);
    atomicAdd(args.cnt_out + 2, cnt.inv); atomicAdd(args.cnt_out + 3, cnt.red);
  }
}

// ---------------------------------------------------------------------------------
// Modular GEMM on CUDA cores: C <- C - A B mod p  (small / skinny shapes).
// 64x64 output tile per CTA, 256 threads, 4x4 outputs per thread, uint64 accumulation
// with a reduction every `kchunk` products (field.py:149-161 delayed reduction).
// ---------------------------------------------------------------------------------
constexpr int SG_BM = 64, SG_BN = 64, SG_BK = 32;

template <bool kSlow>
__global__ void __launch_bounds__(256) simt_gemm_kernel(View c, View a, View b, ModP mp, const int* stop) {
  if (stopped(stop)) return;
  __shared__ uint32_t As[SG_BK][SG_BM + 4];
  __shared__ uint32_t Bs[SG_BK][SG_BN + 4];
  const int m = c.m, n = c.n, k = a.n;
  const int m0 = blockIdx.y * SG_BM, n0 = blockIdx.x * SG_BN;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  uint64_t acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0;
  uint64_t since = 0;
  for (int k0 = 0; k0 < k; k0 += SG_BK) {
    {
      uint32_t va[8], vb[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int idx = tid + q * 256, i = idx / SG_BK, kk = idx % SG_BK;
        const int gi = m0 + i, gk = k0 + kk;
        va[q] = (gi < m && gk < k) ? a.at(gi, gk) : 0u;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int idx = tid + q * 256, kk = idx / SG_BN, j = idx % SG_BN;
        const int gk = k0 + kk, gj = n0 + j;
        vb[q] = (gk < k && gj < n) ? b.at(gk, gj) : 0u;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int idx = tid + q * 256;
        As[idx % SG_BK][idx / SG_BK] = va[q];
        Bs[idx / SG_BN][idx % SG_BN] = vb[q];
      }
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < SG_BK; ++kk) {
      uint32_t av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += (uint64_t)av[i] * bv[j];
      if (kSlow) {
        if (++since == mp.kchunk) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = reduce64(acc[i][j], mp);
          since = 0;
        }
      }
    }
    if (!kSlow) {
      since += SG_BK;
      if (since + SG_BK > mp.kchunk) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = reduce64(acc[i][j], mp);
        since = 0;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int gi = m0 + ty * 4 + i;
    if (gi >= m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int gj = n0 + tx * 4 + j;
      if (gj < n) c.at(gi, gj) = submod(c.at(gi, gj), reduce64(acc[i][j], mp), mp);
    }
  }
}

// ---------------------------------------------------------------------------------
// TRSM (kernels.py:59-120) as "invert the 64x64 diagonal blocks once, then multiply".
// All diagonal-block inverses of a triangular factor are computed in ONE launch
// (one CTA per block), so the recursive TRSM's critical path is only small
// GEMM-shaped kernels; exact arithmetic makes the result identical to substitution.
// ---------------------------------------------------------------------------------
constexpr int TR_BASE = 64;

__device__ __forceinline__ uint32_t acc_dot(const uint32_t* a, int sa, const uint32_t* b, int sb, int k,
                                            const ModP mp) {
  uint64_t acc = 0;
  if ((uint64_t)k <= mp.kchunk) {
    for (int t = 0; t < k; ++t) acc += (uint64_t)a[t * sa] * b[t * sb];
  } else {
    uint64_t c = 0;
    for (int t = 0; t < k; ++t) {
      acc += (uint64_t)a[t * sa] * b[t * sb];
      if (++c == mp.kchunk) { acc = reduce64(acc, mp); c = 0; }
    }
  }
  return reduce64(acc, mp);
}

// Blocked triangular inverse of one 64x64 diagonal block (padded with the identity
// past w): 16x16 diagonal sub-blocks by substitution (thread per column), then two
// merge levels  X12 = -X11 * U12 * X22  (upper)  /  X21 = -X22 * L21 * X11  (lower).
// 256 threads; the serial chain is <= 16 substitution steps instead of 63.
template <bool kUpper>
__device__ void trinv_block(uint32_t (*M)[TR_BASE + 1], uint32_t (*X)[TR_BASE + 1], uint32_t (*T)[33],
                            const uint32_t* dinv, const ModP mp) {
  const int tid = threadIdx.x;
  for (int idx = tid; idx < TR_BASE * TR_BASE; idx += blockDim.x) X[idx >> 6][idx & 63] = 0u;
  __syncthreads();
  if (tid < 64) {  // 4 sub-blocks x 16 columns
    const int b0 = (tid >> 4) * 16, j = tid & 15;
    if (kUpper) {
      X[b0 + j][b0 + j] = dinv[b0 + j];
      for (int i = j - 1; i >= 0; --i) {
        uint64_t acc = 0;
        for (int t = i + 1; t <= j; ++t) acc = acc + (uint64_t)M[b0 + i][b0 + t] * X[b0 + t][b0 + j];
        const uint32_t s = reduce64(acc, mp);
        X[b0 + i][b0 + j] = mulmod(s ? mp.p - s : 0u, dinv[b0 + i], mp);
      }
    } else {
      X[b0 + j][b0 + j] = 1u;
      for (int i = j + 1; i < 16; ++i) {
        uint64_t acc = 0;
        for (int t = j; t < i; ++t) acc = acc + (uint64_t)M[b0 + i][b0 + t] * X[b0 + t][b0 + j];
        const uint32_t s = reduce64(acc, mp);
        X[b0 + i][b0 + j] = s ? mp.p - s : 0u;
      }
    }
  }
  __syncthreads();
  for (int h = 16; h < TR_BASE; h *= 2) {
    // pairs of h x h blocks at offsets b0 (first) and b0 + h (second)
    const int npairs = TR_BASE / (2 * h);
    // T = M12 * X22 (upper)  or  T = M21 * X11 (lower), h x h per pair
    for (int idx = tid; idx < npairs * h * h; idx += blockDim.x) {
      const int pi = idx / (h * h), e = idx % (h * h), i = e / h, j = e % h;
      const int b0 = pi * 2 * h;
      uint64_t acc = 0;
      if (kUpper)
        for (int t = 0; t < h; ++t) acc += (uint64_t)M[b0 + i][b0 + h + t] * X[b0 + h + t][b0 + h + j];
      else
        for (int t = 0; t < h; ++t) acc += (uint64_t)M[b0 + h + i][b0 + t] * X[b0 + t][b0 + j];
      T[pi * h + i][j] = reduce64(acc, mp);  // h <= 32, npairs*h <= 32
    }
    __syncthreads();
    // X12 = -X11 * T (upper)  or  X21 = -X22 * T (lower)
    for (int idx = tid; idx < npairs * h * h; idx += blockDim.x) {
      const int pi = idx / (h * h), e = idx % (h * h), i = e / h, j = e % h;
      const int b0 = pi * 2 * h;
      uint64_t acc = 0;
      if (kUpper)
        for (int t = 0; t < h; ++t) acc += (uint64_t)X[b0 + i][b0 + t] * T[pi * h + t][j];
      else
        for (int t = 0; t < h; ++t) acc += (uint64_t)X[b0 + h + i][b0 + h + t] * T[pi * h + t][j];
      const uint32_t s = reduce64(acc, mp);
      if (kUpper) X[b0 + i][b0 + h + j] = s ? mp.p - s : 0u;
      else X[b0 + h + i][b0 + j] = s ? mp.p - s : 0u;
    }
    __syncthreads();
  }
}

// Products of <= 32 terms stay below 2^64 only when 32 (p-1)^2 < 2^64: p < 2^29.5.
// Larger p (allow_large_modulus) fall back to per-product reduction via the slow path.
__device__ __forceinline__ bool trinv_fast(const ModP mp) { return mp.kchunk >= 32; }

template <bool kUpper>
__device__ void trinv_block_slow(uint32_t (*M)[TR_BASE + 1], uint32_t (*X)[TR_BASE + 1], int w,
                                 const uint32_t* dinv, const ModP mp) {
  // column substitution with per-product reduction (rare: p > 2^29)
  const int j = threadIdx.x;
  if (j < TR_BASE) {
    for (int i = 0; i < TR_BASE; ++i) X[i][j] = 0;
    if (kUpper) {
      X[j][j] = dinv[j];
      for (int i = j - 1; i >= 0; --i) {
        uint64_t acc = 0;
        for (int t = i + 1; t <= j; ++t) acc = reduce64(acc + (uint64_t)M[i][t] * X[t][j], mp);
        X[i][j] = mulmod(acc ? mp.p - (uint32_t)acc : 0u, dinv[i], mp);
      }
    } else {
      X[j][j] = 1;
      for (int i = j + 1; i < TR_BASE; ++i) {
        uint64_t acc = 0;
        for (int t = j; t < i; ++t) acc = reduce64(acc + (uint64_t)M[i][t] * X[t][j], mp);
        X[i][j] = acc ? mp.p - (uint32_t)acc : 0u;
      }
    }
  }
  __syncthreads();
}

// out[b] = inverse of the b-th 64x64 diagonal block of U (upper, nonzero diagonal).
__global__ void __launch_bounds__(256) trinv_upper_kernel(View u, uint32_t* out, ModP mp, const uint16_t* invtab,
                                                          const int* stop) {
  if (stopped(stop)) return;
  __shared__ uint32_t Us[TR_BASE][TR_BASE + 1];
  __shared__ uint32_t X[TR_BASE][TR_BASE + 1];
  __shared__ uint32_t T[32][33];
  __shared__ uint32_t dinv[TR_BASE];
  const int base = blockIdx.x * TR_BASE;
  const int w = min(TR_BASE, u.m - base);
  {
    const int j = threadIdx.x & 63, i0 = threadIdx.x >> 6;  // 4 rows per pass
    uint32_t v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int i = i0 + 4 * q;
      v[q] = (i < w && j < w) ? u.at(base + i, base + j) : (i == j ? 1u : 0u);
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) Us[i0 + 4 * q][j] = v[q];
  }
  __syncthreads();
  if (threadIdx.x < TR_BASE) {
    const uint32_t d = Us[threadIdx.x][threadIdx.x];
    dinv[threadIdx.x] = invtab ? invtab[d] : invmod(d, mp);
  }
  __syncthreads();
  if (trinv_fast(mp)) trinv_block<true>(Us, X, T, dinv, mp);
  else trinv_block_slow<true>(Us, X, w, dinv, mp);
  uint32_t* o = out + (size_t)blockIdx.x * TR_BASE * TR_BASE;
  for (int idx = threadIdx.x; idx < TR_BASE * TR_BASE; idx += blockDim.x) o[idx] = X[idx >> 6][idx & 63];
}

// out[b] = inverse of the b-th diagonal block of unit-lower L (diagonal implicit 1).
__global__ void __launch_bounds__(256) trinv_lower_unit_kernel(View l, uint32_t* out, ModP mp, const int* stop) {
  if (stopped(stop)) return;
  __shared__ uint32_t Ls[TR_BASE][TR_BASE + 1];
  __shared__ uint32_t X[TR_BASE][TR_BASE + 1];
  __shared__ uint32_t T[32][33];
  __shared__ uint32_t dinv[TR_BASE];
  const int base = blockIdx.x * TR_BASE;
  const int w = min(TR_BASE, l.m - base);
  {
    const int j = threadIdx.x & 63, i0 = threadIdx.x >> 6;
    uint32_t v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int i = i0 + 4 * q;
      v[q] = (i < w && j < w && j < i) ? l.at(base + i, base + j) : (i == j ? 1u : 0u);
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) Ls[i0 + 4 * q][j] = v[q];
  }
  if (threadIdx.x < TR_BASE) dinv[threadIdx.x] = 1u;
  __syncthreads();
  if (trinv_fast(mp)) trinv_block<false>(Ls, X, T, dinv, mp);
  else trinv_block_slow<false>(Ls, X, w, dinv, mp);
  uint32_t* o = out + (size_t)blockIdx.x * TR_BASE * TR_BASE;
  for (int idx = threadIdx.x; idx < TR_BASE * TR_BASE; idx += blockDim.x) o[idx] = X[idx >> 6][idx & 63];
}

// 128x128 triangular block: B' = I - T^-1 from the inverses of its two 64x64 diagonal
// blocks (trinv_*_kernel output, 2 x 64 x 64), so that the whole TRSM becomes ONE
// in-place modular GEMM: B U^-1 = B - B (I - U^-1) and L^-1 B = B - (I - L^-1) B (the
// tensor-core GEMM splits its A and B operands into limb planes before the MMA kernel,
// so C may alias either operand).  Off-diagonal block of the inverse:
//   upper  [X1 X12; 0 X2]:  X12 = -X1 (U12 X2)
//   lower  [Y1 0; Y21 Y2]:  Y21 = -Y2 (L21 Y1)
// Grid: 4 CTAs, each writes 32 columns of B'; the two CTAs over the off-diagonal block
// compute their 32 columns of it (2 x 64 x 32 x 64 MACs).
template <bool kUpper>
__global__ void __launch_bounds__(256) trinv128_combine_kernel(View t, const uint32_t* inv64, uint32_t* bp,
                                                               ModP mp, const int* stop, int ldb = 128) {
  if (stopped(stop)) return;
  __shared__ uint32_t MA[64][65], M3[64][33], T[64][33];  // MA holds B in pass 0, A in pass 1
  const int tid = threadIdx.x, c0 = 32 * blockIdx.x;  // output columns [c0, c0 + 32)
  const uint32_t* X1 = inv64;                // upper: X1 (top-left); lower: Y1
  const uint32_t* X2 = inv64 + 64 * 64;      // upper: X2 (bottom-right); lower: Y2
  const bool offdiag = kUpper ? c0 >= 64 : c0 < 64;
  if (!offdiag) {
    // diagonal-block columns: I - X (the other block row is 0 - 0 = 0)
    const uint32_t* X = kUpper ? X1 : X2;
    const int cb = kUpper ? c0 : c0 - 64;    // column inside the diagonal block
    const int r0 = kUpper ? 0 : 64;          // block row holding the diagonal block
    for (int idx = tid; idx < 128 * 32; idx += 256) {
      const int i = idx >> 5, j = idx & 31;
      uint32_t v = 0u;
      if (i >= r0 && i < r0 + 64) {
        const uint32_t x = X[(i - r0) * 64 + cb + j];
        const uint32_t d = (i - r0 == cb + j) ? 1u : 0u;
        v = d >= x ? d - x : d + (mp.p - x);
      }
      bp[i * ldb + c0 + j] = v;
    }
    return;
  }
  // off-diagonal columns: Z[:, cols] = -A (B C[:, cols]) with
  //   upper: A = X1, B = U12 = t[0:64, 64:128], C = X2, cols = c0 - 64 ..
  //   lower: A = Y2, B = L21 = t[64:128, 0:64], C = Y1, cols = c0 ..
  const int cc = kUpper ? c0 - 64 : c0;
  const uint32_t* Am = kUpper ? X1 : X2;
  const uint32_t* Cm = kUpper ? X2 : X1;
  for (int idx = tid; idx < 64 * 64; idx += 256) {
    const int i = idx >> 6, j = idx & 63;
    MA[i][j] = kUpper ? t.at(i, 64 + j) : t.at(64 + i, j);
  }
  for (int idx = tid; idx < 64 * 32; idx += 256) {
    const int i = idx >> 5, j = idx & 31;
    M3[i][j] = Cm[i * 64 + cc + j];
  }
  __syncthreads();
  const bool lazy = mp.kchunk >= 64;
  const int i0 = tid >> 3, j0 = (tid & 7) * 4;  // 2 rows x 4 columns per thread: rows i0, i0 + 32
  for (int pass = 0; pass < 2; ++pass) {
    unsigned long long acc[2][4] = {};
    for (int k = 0; k < 64; ++k) {
      const uint32_t a0 = MA[i0][k];
      const uint32_t a1 = MA[i0 + 32][k];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t b = pass == 0 ? M3[k][j0 + q] : T[k][j0 + q];
        acc[0][q] += (unsigned long long)a0 * b;
        acc[1][q] += (unsigned long long)a1 * b;
        if (!lazy) { acc[0][q] = reduce64(acc[0][q], mp); acc[1][q] = reduce64(acc[1][q], mp); }
      }
    }
    if (pass == 0) {
#pragma unroll
      for (int q = 0; q < 4; ++q) { T[i0][j0 + q] = reduce64(acc[0][q], mp); T[i0 + 32][j0 + q] = reduce64(acc[1][q], mp); }
      __syncthreads();  // every read of MA (= B) is done
      for (int idx = tid; idx < 64 * 64; idx += 256) MA[idx >> 6][idx & 63] = Am[idx];
      __syncthreads();
    } else {
      // B' = I - Inv = -Z = A (B C) on the off-diagonal block (its identity part is 0)
      const int rb = kUpper ? 0 : 64;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        bp[(rb + i0) * ldb + c0 + j0 + q] = reduce64(acc[0][q], mp);
        bp[(rb + i0 + 32) * ldb + c0 + j0 + q] = reduce64(acc[1][q], mp);
      }
    }
  }
  // the diagonal block in these columns: I - X2 (upper, rows 64..127) or I - Y1 (lower, rows 0..63)
  {
    const int rb = kUpper ? 64 : 0;          // block row of the diagonal block in these columns
    const uint32_t* X = kUpper ? X2 : X1;
    for (int idx = tid; idx < 64 * 32; idx += 256) {
      const int i = idx >> 5, j = idx & 31;
      const uint32_t x = X[i * 64 + cc + j];
      const uint32_t d = (i == cc + j) ? 1u : 0u;
      bp[(rb + i) * ldb + c0 + j] = d >= x ? d - x : d + (mp.p - x);
    }
  }
}

// B <- B * Uinv for a w-column block (w <= 64): one CTA owns 32 rows of B (in place);
// 128 threads, each a 4x4 register tile (8 shared loads per 16 products).
__global__ void __launch_bounds__(128) trsm_apply_right_kernel(View b, const uint32_t* uinv, ModP mp,
                                                               const int* stop) {
  if (stopped(stop)) return;
  __shared__ uint32_t Bs[32][TR_BASE + 4];
  __shared__ uint32_t Ui[TR_BASE][TR_BASE + 4];
  const int w = b.n, r0 = blockIdx.x * 32, rows = min(32, b.m - r0);
  {
    // all staging loads issued back to back (32 + 16 per thread), then stored
    uint32_t u[32], bb[16];
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int idx = threadIdx.x + q * 128, i = idx >> 6, j = idx & 63;
      u[q] = (i < w && j < w) ? __ldg(uinv + i * TR_BASE + j) : 0u;
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int i = (threadIdx.x >> 5) + 4 * (q >> 1), j = (threadIdx.x & 31) + 32 * (q & 1);
      bb[q] = (i < rows && j < w) ? b.at(r0 + i, j) : 0u;
    }
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int idx = threadIdx.x + q * 128;
      Ui[idx >> 6][idx & 63] = u[q];
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) Bs[(threadIdx.x >> 5) + 4 * (q >> 1)][(threadIdx.x & 31) + 32 * (q & 1)] = bb[q];
  }
  __syncthreads();
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;  // rows 4*ty.., cols 4*tx..
  uint64_t acc[4][4] = {};
  const bool fast = mp.kchunk >= TR_BASE;
  for (int t = 0; t < w; ++t) {
    uint32_t av[4], bv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) { av[q] = Bs[4 * ty + q][t]; bv[q] = Ui[t][4 * tx + q]; }
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        acc[x][y] += (uint64_t)av[x] * bv[y];
        if (!fast) acc[x][y] = reduce64(acc[x][y], mp);
      }
  }
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int rr = 4 * ty + x, cc = 4 * tx + y;
      if (rr < rows && cc < w) b.at(r0 + rr, cc) = reduce64(acc[x][y], mp);
    }
}

// B <- Linv * B for a w-row block (w <= 64): one CTA owns 32 columns of B (in place).
__global__ void __launch_bounds__(128) trsm_apply_left_kernel(const uint32_t* linv, View b, ModP mp,
                                                              const int* stop) {
  if (stopped(stop)) return;
  __shared__ uint32_t Bs[TR_BASE][32 + 4];
  __shared__ uint32_t Li[TR_BASE][TR_BASE + 4];
  const int w = b.m, c0 = blockIdx.x * 32, cols = min(32, b.n - c0);
  {
    uint32_t u[32], bb[16];
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int idx = threadIdx.x + q * 128, i = idx >> 6, j = idx & 63;
      u[q] = (i < w && j < w) ? __ldg(linv + i * TR_BASE + j) : 0u;
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int i = (threadIdx.x >> 5) + 4 * q, j = threadIdx.x & 31;
      bb[q] = (i < w && j < cols) ? b.at(i, c0 + j) : 0u;
    }
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int idx = threadIdx.x + q * 128;
      Li[idx >> 6][idx & 63] = u[q];
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) Bs[(threadIdx.x >> 5) + 4 * q][threadIdx.x & 31] = bb[q];
  }
  __syncthreads();
  const int ty = threadIdx.x >> 3, tx = threadIdx.x & 7;  // rows 4*ty.. (64), cols 4*tx.. (32)
  uint64_t acc[4][4] = {};
  const bool fast = mp.kchunk >= TR_BASE;
  for (int t = 0; t < w; ++t) {
    uint32_t av[4], bv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) { av[q] = Li[4 * ty + q][t]; bv[q] = Bs[t][4 * tx + q]; }
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        acc[x][y] += (uint64_t)av[x] * bv[y];
        if (!fast) acc[x][y] = reduce64(acc[x][y], mp);
      }
  }
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int rr = 4 * ty + x, cc = 4 * tx + y;
      if (rr < w && cc < cols) b.at(rr, c0 + cc) = reduce64(acc[x][y], mp);
    }
}

// Full-inverse assembly for the large-triangle TRSM (Ops::tri_inverse / trsm_big_tc).
// place_blocks: the 64 x 64 diagonal-block inverses onto the diagonal of X (clipped at r).
__global__ void place_blocks_kernel(const uint32_t* inv, View x, const int* stop) {
  if (stopped(stop)) return;
  const int b0 = blockIdx.x * TR_BASE, w = min(TR_BASE, x.m - b0);
  const uint32_t* src = inv + (size_t)blockIdx.x * TR_BASE * TR_BASE;
  for (int idx = threadIdx.x; idx < TR_BASE * TR_BASE; idx += blockDim.x) {
    const int i = idx >> 6, j = idx & 63;
    if (i < w && j < w) x.at(b0 + i, b0 + j) = src[idx];
  }
}
__global__ void negate_kernel(View v, ModP mp, const int* stop) {
  if (stopped(stop)) return;
  for (int i = blockIdx.y; i < v.m; i += gridDim.y)
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < v.n; j += gridDim.x * blockDim.x) {
      const uint32_t a = v.at(i, j);
      v.at(i, j) = a ? mp.p - a : 0u;
    }
}
// X <- I - X on the triangle of X (lower: strictly below the diagonal, whose diagonal is 1;
// upper: the diagonal and above), zeros elsewhere are kept.
__global__ void i_minus_kernel(View x, int upper, ModP mp, const int* stop) {
  if (stopped(stop)) return;
  for (int i = blockIdx.y; i < x.m; i += gridDim.y)
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < x.n; j += gridDim.x * blockDim.x) {
      const uint32_t a = x.at(i, j);
      const uint32_t neg = a ? mp.p - a : 0u;
      if (i == j) x.at(i, j) = upper ? (neg + 1u == mp.p ? 0u : neg + 1u) : 0u;
      else x.at(i, j) = neg;
    }
}

// flag <- 1 if any diagonal entry of U is zero (kernels.py:93-95).
__global__ void diag_zero_kernel(View u, int* flag) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < u.m; j += gridDim.x * blockDim.x)
    if (u.at(j, j) == 0u) atomicOr(flag, 1);
}

// ---------------------------------------------------------------------------------
// Permutations restricted to the moved set: tmp[q] <- X[src[q]], then X[dst[q]] <- tmp[q].
// ---------------------------------------------------------------------------------
// Whole-row copies: 16-byte accesses when every row of the view and of the temporary is
// 16-byte aligned (pitch and width multiples of 4), else scalar.
__device__ __forceinline__ void copy_row(uint32_t* d, const uint32_t* s, int n, bool vec) {
  if (vec) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n / 4; j += gridDim.x * blockDim.x)
      reinterpret_cast<uint4*>(d)[j] = reinterpret_cast<const uint4*>(s)[j];
  } else {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) d[j] = s[j];
  }
}
__global__ void rows_to_tmp_kernel(View x, const int* src, int nmv, uint32_t* tmp) {
  const bool vec = (x.ld % 4) == 0 && (x.n % 4) == 0 && (reinterpret_cast<uintptr_t>(x.a) & 15) == 0;
  for (int q = blockIdx.y; q < nmv; q += gridDim.y) copy_row(tmp + (int64_t)q * x.n, x.row(src[q]), x.n, vec);
}
__global__ void tmp_to_rows_kernel(View x, const int* dst, int nmv, const uint32_t* tmp) {
  const bool vec = (x.ld % 4) == 0 && (x.n % 4) == 0 && (reinterpret_cast<uintptr_t>(x.a) & 15) == 0;
  for (int q = blockIdx.y; q < nmv; q += gridDim.y) copy_row(x.row(dst[q]), tmp + (int64_t)q * x.n, x.n, vec);
}
__global__ void cols_to_tmp_kernel(View x, const int* src, int nmv, uint32_t* tmp) {
  for (int i = blockIdx.y; i < x.m; i += gridDim.y) {
    const uint32_t* xr = x.row(i);
    uint32_t* tr = tmp + (int64_t)i * nmv;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nmv; q += gridDim.x * blockDim.x) tr[q] = xr[src[q]];
  }
}
__global__ void tmp_to_cols_kernel(View x, const int* dst, int nmv, const uint32_t* tmp) {
  for (int i = blockIdx.y; i < x.m; i += gridDim.y) {
    uint32_t* xr = x.row(i);
    const uint32_t* tr = tmp + (int64_t)i * nmv;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nmv; q += gridDim.x * blockDim.x) xr[dst[q]] = tr[q];
  }
}

// Row gather in ONE pass for small moved sets (the exact recursion's many small gathers): each
// CTA owns strips of 32 columns, stages the moved rows' 128-byte segments in shared memory and
// writes them back permuted — one launch, no temporary.
__global__ void __launch_bounds__(256) rows_inplace_kernel(View x, const int* __restrict__ src,
                                                           const int* __restrict__ dst, int nmv) {
  extern __shared__ __align__(16) uint32_t s_seg[];  // [nmv][32]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int c0 = blockIdx.x * 32; c0 < x.n; c0 += gridDim.x * 32) {
    const int col = c0 + lane;
    if (col < x.n)
      for (int q = w; q < nmv; q += 8) s_seg[q * 32 + lane] = x.at(src[q], col);
    __syncthreads();
    if (col < x.n)
      for (int q = w; q < nmv; q += 8) x.at(dst[q], col) = s_seg[q * 32 + lane];
    __syncthreads();
  }
}

// Column gather in ONE pass, in place: the moved set of a column permutation is closed, so a
// row's moved entries all lie in the column span [lo, lo + span).  Each CTA stages that span
// of a row in shared memory (cp.async, 16-byte chunks where the row is aligned; the next row
// is prefetched into the other buffer when two fit) and writes X[i, dst[q]] <- row[src[q]]
// back over it: HBM traffic is one read and one write of the span instead of the two
// scattered passes through a temporary (cols_to_tmp / tmp_to_cols).
__global__ void __launch_bounds__(1024, 1) cols_inplace_kernel(View x, const int* __restrict__ src,
                                                               const int* __restrict__ dst, int nmv, int lo,
                                                               int span, int nbuf) {
  extern __shared__ __align__(16) uint32_t s_rows[];
  // buffers are padded so that a row's 16-byte-aligned global chunks land 16-byte aligned
  const int pitch = (span + 3) / 4 * 4 + 8;
  auto stage = [&](int i, int b) {
    const uint32_t* g = x.row(i) + lo;
    const int mis = (int)((reinterpret_cast<uintptr_t>(g) >> 2) & 3);  // words past a 16-byte boundary
    uint32_t* s = s_rows + (size_t)b * pitch + mis;                    // same misalignment in shared memory
    const int head = min(span, (4 - mis) & 3);
    const int body = (span - head) / 4;
    for (int j = threadIdx.x; j < body; j += blockDim.x) {
      const unsigned sa = (unsigned)__cvta_generic_to_shared(s + head + 4 * j);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g + head + 4 * j));
    }
    const int tail0 = head + 4 * body;
    for (int j = threadIdx.x; j < head + (span - tail0); j += blockDim.x) {
      const int e = j < head ? j : tail0 + (j - head);
      const unsigned sa = (unsigned)__cvta_generic_to_shared(s + e);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(g + e));
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  int i = blockIdx.x, b = 0;
  if (i < x.m) stage(i, 0);
  for (; i < x.m; i += gridDim.x) {
    const int nx = i + gridDim.x;
    if (nbuf == 2 && nx < x.m) {
      stage(nx, b ^ 1);
      asm volatile("cp.async.wait_group 1;\n" ::);
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncthreads();
    uint32_t* g = x.row(i);
    const int mis = (int)((reinterpret_cast<uintptr_t>(g + lo) >> 2) & 3);
    const uint32_t* s = s_rows + (size_t)b * pitch + mis - lo;
    for (int q = threadIdx.x; q < nmv; q += blockDim.x) g[dst[q]] = s[src[q]];
    __syncthreads();  // the buffer is free again
    if (nbuf == 2) b ^= 1;
    else if (nx < x.m) stage(nx, 0);
  }
}

// ---------------------------------------------------------------------------------
// Un-factoring (Driver::unfactor): re-multiplying partial factors in place, so that a failed
// speculative LU restores its node without a backup copy of the whole matrix.
// ---------------------------------------------------------------------------------
// Dense 64 x 64 copy (pitch TR_BASE) of a triangle of t (w <= 64): upper = 1 keeps i <= j,
// upper = 0 keeps i > j and puts 1 on the diagonal (unit lower); zeros elsewhere.
__global__ void tri_extract_kernel(View t, uint32_t* out, int upper) {
  const int w = t.m;
  for (int idx = threadIdx.x; idx < TR_BASE * TR_BASE; idx += blockDim.x) {
    const int i = idx >> 6, j = idx & 63;
    uint32_t v = 0u;
    if (i < w && j < w) {
      if (upper) v = i <= j ? t.at(i, j) : 0u;
      else v = i > j ? t.at(i, j) : (i == j ? 1u : 0u);
    }
    out[idx] = v;
  }
}
// X (w x w, w <= 64, packed unit-lower L below the diagonal and U on/above it) <- L U, one CTA.
__global__ void __launch_bounds__(256) lu_mult_kernel(View x, ModP mp) {
  __shared__ uint32_t S[TR_BASE][TR_BASE + 1];
  const int w = x.m;
  for (int idx = threadIdx.x; idx < w * w; idx += blockDim.x) S[idx / w][idx % w] = x.at(idx / w, idx % w);
  __syncthreads();
  const bool fast = mp.kchunk >= TR_BASE + 1;
  for (int idx = threadIdx.x; idx < w * w; idx += blockDim.x) {
    const int i = idx / w, j = idx % w, kmax = min(i, j);  // sum over k < min(i, j), then the k = min term
    unsigned long long acc = 0;
    for (int k = 0; k < kmax; ++k) {
      acc += (unsigned long long)S[i][k] * S[k][j];
      if (!fast) acc = reduce64(acc, mp);
    }
    // k = min(i, j): L[i][i] = 1 when i <= j, else L[i][j] U[j][j]
    acc += i <= j ? (unsigned long long)S[i][j] : (unsigned long long)S[i][j] * S[j][j];
    x.at(i, j) = reduce64(acc, mp);
  }
}

// *out <- min(*out, smallest column of a nonzero in row 0 of x) (pivot repair of the
// speculative LU: row-order elimination picks the leftmost nonzero, pluq_rpm.cuh phase a).
__global__ void first_nonzero_kernel(View x, int* out) {
  int best = 0x7fffffff;
  const uint32_t* r = x.row(0);
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < x.n; j += gridDim.x * blockDim.x)
    if (r[j] != 0u) { best = j; break; }
  for (int o = 16; o; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0 && best != 0x7fffffff) atomicMin(out, best);
}

// flag <- 1 if the block holds any nonzero (zero-block short-circuit).
// 16-byte loads when rows allow it; blocks stop early once any block has set the flag (a
// nonzero Schur complement is usually nonzero right at its first rows).
__global__ void nonzero_kernel(View x, int* flag) {
  bool nz = false;
  const bool vec = (x.ld % 4) == 0 && (reinterpret_cast<uintptr_t>(x.a) & 15) == 0;
  const int n4 = vec ? x.n / 4 : 0;
  for (int i = blockIdx.y; i < x.m; i += gridDim.y) {
    const uint32_t* xr = x.row(i);
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n4; j += gridDim.x * blockDim.x) {
      const uint4 q = reinterpret_cast<const uint4*>(xr)[j];
      nz |= (q.x | q.y | q.z | q.w) != 0u;
    }
    for (int j = 4 * n4 + blockIdx.x * blockDim.x + threadIdx.x; j < x.n; j += gridDim.x * blockDim.x) nz |= xr[j] != 0u;
    if (((i - blockIdx.y) / gridDim.y & 7) == 7) {  // every 8 rows: stop if anyone found a nonzero
      if (__syncthreads_or(nz) || *reinterpret_cast<volatile int*>(flag)) {
        if (threadIdx.x == 0) atomicOr(flag, 1);
        return;
      }
    }
  }
  if (__syncthreads_or(nz) && threadIdx.x == 0) atomicOr(flag, 1);
}

// Compact node backup (p < 2^16): residues stored as uint16, rows packed (pitch = n).
// 16-byte loads / 8-byte stores when the rows allow it (HBM-bound: 6 bytes per entry).
__device__ __forceinline__ bool rows16_vec(const View& v) {
  return (v.ld % 4) == 0 && (v.n % 4) == 0 && (reinterpret_cast<uintptr_t>(v.a) & 15) == 0;
}
// With `bad`, the copy doubles as the input range check (entries >= p set *bad), so a large
// node's validation costs no extra read of the matrix.
__global__ void copy_to16_kernel(uint16_t* dst, View src, uint32_t p, int* bad) {
  bool b = false;
  if (rows16_vec(src)) {
    const int64_t nq = src.n / 4, total = (int64_t)src.m * nq;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
      const int64_t i = t / nq, q = t - i * nq;
      const uint4 v = reinterpret_cast<const uint4*>(src.a + i * src.ld)[q];
      b |= (v.x >= p) | (v.y >= p) | (v.z >= p) | (v.w >= p);
      reinterpret_cast<uint2*>(dst + i * src.n)[q] = make_uint2(v.x | (v.y << 16), v.z | (v.w << 16));
    }
  } else {
    const int64_t total = (int64_t)src.m * src.n;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
      const int64_t i = t / src.n, j = t - i * src.n;
      const uint32_t v = src.a[i * src.ld + j];
      b |= v >= p;
      dst[t] = (uint16_t)v;
    }
  }
  if (bad && __syncthreads_or(b) && threadIdx.x == 0) atomicOr(bad, 1);
}
__global__ void backup32_kernel(uint32_t* dst, View src, uint32_t p, int* bad) {
  bool b = false;
  const int64_t total = (int64_t)src.m * src.n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / src.n, j = t - i * src.n;
    const uint32_t v = src.a[i * src.ld + j];
    b |= v >= p;
    dst[t] = v;
  }
  if (bad && __syncthreads_or(b) && threadIdx.x == 0) atomicOr(bad, 1);
}
__global__ void copy_from16_kernel(View dst, const uint16_t* src) {
  if (rows16_vec(dst)) {
    const int64_t nq = dst.n / 4, total = (int64_t)dst.m * nq;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
      const int64_t i = t / nq, q = t - i * nq;
      const uint2 v = reinterpret_cast<const uint2*>(src + i * dst.n)[q];
      reinterpret_cast<uint4*>(dst.a + i * dst.ld)[q] = make_uint4(v.x & 0xffffu, v.x >> 16, v.y & 0xffffu, v.y >> 16);
    }
    return;
  }
  const int64_t total = (int64_t)dst.m * dst.n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / dst.n, j = t - i * dst.n;
    dst.a[i * dst.ld + j] = src[t];
  }
}

__global__ void copy_view_kernel(View dst, View src) {
  for (int i = blockIdx.y; i < dst.m; i += gridDim.y)
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < dst.n; j += gridDim.x * blockDim.x)
      dst.at(i, j) = src.at(i, j);
}

// 32-bit table of inverses for 2^16 <= p <= 2^25 (ModP::itab32): tab[a] = a^-1, tab[0] = 0.
// mp must come without a table (Euclid builds it).
__global__ void invtab32_kernel(uint32_t* tab, ModP mp) {
  for (uint32_t a = blockIdx.x * blockDim.x + threadIdx.x; a < mp.p; a += gridDim.x * blockDim.x)
    tab[a] = a ? invmod(a, mp) : 0u;
}

// Table of inverses mod p (p < 2^16): tab[a] = a^-1, tab[0] = 0.
__global__ void invtab_kernel(uint16_t* tab, ModP mp) {
  for (uint32_t a = blockIdx.x * blockDim.x + threadIdx.x; a < mp.p; a += gridDim.x * blockDim.x)
    tab[a] = a ? (uint16_t)invmod(a, mp) : 0;
}

// Diagonal block of the speculative LU, latency-optimised (one CTA of 1024 threads,
// block <= 128 x 128): Crout with every dot product split over 4 threads (shuffle
// reduction), the pivot settled first (a zero pivot leaves row/column t untouched for
// the host finish), and the pivot inverse from a shared-memory copy of the inverse
// table when p < 2^16.
__global__ void __launch_bounds__(1024) diag_crout_fast_kernel(View blk, ModP mp, const uint16_t* invtab, int* stop,
                                                              int* status, int k0) {
  if (stopped(stop)) return;
  extern __shared__ __align__(16) uint32_t smem_dyn[];
  const int m = blk.m, n = blk.n, mn = min(m, n), lds = n | 1;
  const int tid = threadIdx.x, nt = blockDim.x;
  uint32_t* A = smem_dyn;
  uint16_t* tab = reinterpret_cast<uint16_t*>(smem_dyn + ((m * lds + 3) & ~3));
  const bool use_tab = invtab != nullptr;
  if (use_tab) {
    const int words = (int)(mp.p + 1) / 2;
    const uint4* src = reinterpret_cast<const uint4*>(invtab);
    uint4* dst = reinterpret_cast<uint4*>(tab);
    for (int q = tid; q < (words + 3) / 4; q += nt) dst[q] = __ldg(src + q);
  }
  for (int idx = tid; idx < m * n; idx += nt) {
    const int i = idx / n, j = idx - (idx / n) * n;
    A[i * lds + j] = blk.at(i, j);
  }
  __syncthreads();
  const int sub = tid & 3, item0 = tid >> 2;
  const bool fast = mp.kchunk >= 40;  // <= 32 products per partial sum without reduction
  int stop_t = mn;
  for (int t = 0; t < mn; ++t) {
    // phase A: U row t (j >= t, incl. the pivot) and L column t numerators (i > t),
    // 4 threads per dot product; each writer keeps its dot product to undo on a zero pivot
    const int nu = n - t, nl = m - t - 1;
    const int q = item0;  // nu + nl <= 255 < 256 items per pass
    const bool live = q < nu + nl;
    const int i = q < nu ? t : t + 1 + (q - nu);
    const int j = q < nu ? t + q : t;
    uint64_t acc = 0;
    if (live) {
      const uint32_t* li = A + i * lds;
      if (fast) {
        int kk = sub;
        for (; kk + 12 < t; kk += 16) {
          acc += (uint64_t)li[kk] * A[kk * lds + j];
          acc += (uint64_t)li[kk + 4] * A[(kk + 4) * lds + j];
          acc += (uint64_t)li[kk + 8] * A[(kk + 8) * lds + j];
          acc += (uint64_t)li[kk + 12] * A[(kk + 12) * lds + j];
        }
        for (; kk < t; kk += 4) acc += (uint64_t)li[kk] * A[kk * lds + j];
      } else {
        for (int kk = sub; kk < t; kk += 4) acc = reduce64(acc + (uint64_t)li[kk] * A[kk * lds + j], mp);
      }
    }
    uint32_t v = reduce64(acc, mp);
    v = addmod(v, __shfl_xor_sync(0xffffffffu, v, 1), mp);
    v = addmod(v, __shfl_xor_sync(0xffffffffu, v, 2), mp);
    const bool writer = live && sub == 0;
    if (writer) A[i * lds + j] = submod(A[i * lds + j], v, mp);
    __syncthreads();
    const uint32_t piv = A[t * lds + t];
    if (piv == 0u) {
      // zero pivot: undo phase A so row t / column t are untouched for the host finish
      if (writer) A[i * lds + j] = addmod(A[i * lds + j], v, mp);
      stop_t = t;
      break;
    }
    // phase B: scale the L column by the pivot inverse
    const uint32_t inv = use_tab ? (uint32_t)tab[piv] : invmod(piv, mp);
    if (writer && q >= nu) A[i * lds + j] = mulmod(A[i * lds + j], inv, mp);
    __syncthreads();
  }
  __syncthreads();
  for (int idx = tid; idx < m * n; idx += nt) {
    const int i = idx / n, j = idx - (idx / n) * n;
    blk.at(i, j) = A[i * lds + j];
  }
  if (tid == 0 && stop_t < mn) {
    status[0] = k0;
    status[1] = stop_t;
    __threadfence();
    atomicExch(stop, 1);
  }
}

// Right-looking lazy-reduction variant of diag_crout_fast_kernel, same contract: the
// block (m, n <= 128) is factored in place; on a zero pivot at t the entries with
// i < t or j < t hold the factors of the first t pivots, the trailing block keeps its
// original values, and (status, stop) report (k0, t).  Warp w holds rows 4w..4w+3,
// lane l columns l + 32q (q < 4), every element in a 64-bit register accumulator that
// takes one IMAD.WIDE per pivot; elements are reduced mod p once, when they become
// part of pivot row t (U) or column t (L).  For primes where 128 products no longer fit
// in 64 bits, all accumulators are reduced every kchunk - 1 steps.
template <int RW>  // rows per warp: 4 (32 warps) or 8 (16 warps, no register pressure)
__global__ void __launch_bounds__(32 * (128 / RW)) diag_lazy_kernel(View blk, ModP mp, const uint16_t* invtab,
                                                                    int* stop, int* status, int k0) {
  constexpr int NT = 32 * (128 / RW);
  if (stopped(stop)) return;
  extern __shared__ __align__(16) uint32_t smem_dyn[];
  constexpr int B = 128, LD = B + 1;
  const int m = blk.m, n = blk.n, mn = min(m, n);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const bool use_tab = invtab != nullptr;
  uint16_t* tab = reinterpret_cast<uint16_t*>(smem_dyn);     // inverse table first (16-byte aligned)
  unsigned long long* mbuf = reinterpret_cast<unsigned long long*>(smem_dyn + (use_tab ? 32768 : 0));  // [NW][RW]
  uint32_t* lbuf = reinterpret_cast<uint32_t*>(mbuf + 128);     // [NW][RW]
  uint32_t* pinv = lbuf + 128;                                  // [2]
  uint32_t* prow = pinv + 2;                                    // [2][B] pivot rows
  uint32_t* out = prow + 2 * B;                                 // [B][LD] output image
  if (use_tab) {
    const int words = (int)(mp.p + 1) / 2;
    const uint4* src = reinterpret_cast<const uint4*>(invtab);
    uint4* dst = reinterpret_cast<uint4*>(tab);
    for (int q = tid; q < (words + 3) / 4; q += NT) dst[q] = __ldg(src + q);
  }
  const int r0 = RW * w;
  unsigned long long acc[RW][4];
#pragma unroll
  for (int rr = 0; rr < RW; ++rr)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = r0 + rr, j = lane + 32 * q;
      const uint32_t v = (i < m && j < n) ? blk.at(i, j) : 0u;
      acc[rr][q] = v;
      if (i < m && j < n) out[i * LD + j] = v;
    }
  __syncthreads();  // the table is in shared memory
  auto pivinv = [&](uint32_t d) -> uint32_t { return d ? (use_tab ? (uint32_t)tab[d] : invmod(d, mp)) : 0u; };
  if (w == 0) {  // row 0 is final from the start
#pragma unroll
    for (int q = 0; q < 4; ++q) prow[lane + 32 * q] = (uint32_t)acc[0][q];
    if (lane == 0) pinv[0] = mn > 0 ? pivinv((uint32_t)acc[0][0]) : 0u;
  }
  const uint64_t kc1 = mp.kchunk > 1 ? mp.kchunk - 1 : 1;
  const int kred = kc1 > (1u << 20) ? (1 << 20) : (int)kc1;
  int since = 0, stop_t = mn;
#ifdef PLUQ_TRACE
  long long T[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const bool trw = k0 == 0 && (tid >> 5) == (64 / RW);  // owner warp of row 64
#define DMARK(x) do { if (trw && t == 63 && lane == 0) T[x] = clock64(); } while (0)
#else
#define DMARK(x) do { } while (0)
#endif
  for (int t = 0; t < mn; ++t) {
    DMARK(0);
    __syncthreads();  // pivot row t published
    DMARK(1);
    const uint32_t iv = pinv[t & 1];
    if (iv == 0u) { stop_t = t; break; }  // block-uniform
    uint32_t nrv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t u = prow[(t & 1) * B + lane + 32 * q];
      nrv[q] = (lane + 32 * q > t && u) ? mp.p - u : 0u;  // columns <= t take no update
    }
    if (r0 + RW - 1 > t && r0 < m) {  // warp has rows below the pivot (warp-uniform)
      const int tq = t >> 5;
      if (lane == (t & 31)) {
#pragma unroll
        for (int rr = 0; rr < RW; ++rr) {
          unsigned long long x = acc[rr][0];
#pragma unroll
          for (int q = 1; q < 4; ++q) x = q == tq ? acc[rr][q] : x;
          mbuf[w * RW + rr] = x;
        }
      }
      __syncwarp();
      DMARK(2);
      if (lane < RW) {
        const int i = r0 + lane;
        uint32_t l = 0u;
        if (i > t && i < m) {
          l = mulmod(reduce64(mbuf[w * RW + lane], mp), iv, mp);
          out[i * LD + t] = l;  // L entry, final
        }
        lbuf[w * RW + lane] = l;
      }
      __syncwarp();
      DMARK(3);
#pragma unroll
      for (int rr = 0; rr < RW; ++rr) {
        const uint32_t l = lbuf[w * RW + rr];
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[rr][q] += (unsigned long long)l * nrv[q];
      }
    }
    if (++since >= kred) {  // large p: keep the accumulators in range (block-uniform)
      since = 0;
#pragma unroll
      for (int rr = 0; rr < RW; ++rr)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[rr][q] = reduce64(acc[rr][q], mp);
    }
    DMARK(4);
    const int t1 = t + 1;  // row t+1 is final: its owner reduces and publishes it
    if (t1 < mn && t1 / RW == w) {
      const int rr1 = t1 % RW;
      uint32_t x[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        unsigned long long y = acc[0][q];
#pragma unroll
        for (int rr = 1; rr < RW; ++rr) y = rr == rr1 ? acc[rr][q] : y;
        x[q] = reduce64(y, mp);
      }
      const uint32_t d = __shfl_sync(0xffffffffu, lane_pick<4>(x, t1 >> 5), t1 & 31);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = lane + 32 * q;
        prow[(t1 & 1) * B + c] = c >= t1 && c < n ? x[q] : 0u;
        if (d != 0u && c >= t1 && c < n) out[t1 * LD + c] = x[q];  // U row (kept original on a zero pivot)
      }
      if (lane == 0) pinv[t1 & 1] = pivinv(d);
    }
    DMARK(5);
#ifdef PLUQ_TRACE
    if (trw && t == 63 && lane == 0)
      printf("DIAG t=63 bar=%lld mul_stage=%lld mult=%lld imad=%lld fin=%lld total_to_bar=%lld\n", T[1] - T[0],
             T[2] - T[1], T[3] - T[2], T[4] - T[3], T[5] - T[4], T[5] - T[1]);
#endif
  }
  __syncthreads();
  for (int idx = tid; idx < m * n; idx += NT) {
    const int i = idx / n, j = idx - (idx / n) * n;
    blk.at(i, j) = out[i * LD + j];
  }
  if (tid == 0 && stop_t < mn) {
    status[0] = k0;
    status[1] = stop_t;
    __threadfence();
    atomicExch(stop, 1);
  }
}

inline size_t diag_lazy_smem(bool tab) {
  return (size_t)(128 * 129 + 2 * 128 + 2) * 4 + 128 * 8 + 128 * 4 + 16 + (tab ? 65536 * 2 : 0);
}

inline size_t diag_fast_smem(int64_t bs, bool tab) {
  return (size_t)(((bs * (bs | 1)) + 3) & ~3ll) * 4 + (tab ? 65536 * 2 : 0);
}

// uint16 wire of the host pipeline (p <= 2^16): widen / narrow, 8 entries per iteration
// with 16-byte accesses (chunks start at multiples of the chunk size: aligned).
__global__ void widen16_kernel(const uint16_t* in, uint32_t* out, int64_t count) {
  const int64_t n8 = count / 8;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n8; t += (int64_t)gridDim.x * blockDim.x) {
    const uint4 v = reinterpret_cast<const uint4*>(in)[t];
    reinterpret_cast<uint4*>(out)[2 * t] = make_uint4(v.x & 0xffffu, v.x >> 16, v.y & 0xffffu, v.y >> 16);
    reinterpret_cast<uint4*>(out)[2 * t + 1] = make_uint4(v.z & 0xffffu, v.z >> 16, v.w & 0xffffu, v.w >> 16);
  }
  for (int64_t t = 8 * n8 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = in[t];
}
__global__ void narrow16_kernel(const uint32_t* in, uint16_t* out, int64_t count) {
  const int64_t n8 = count / 8;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n8; t += (int64_t)gridDim.x * blockDim.x) {
    const uint4 a = reinterpret_cast<const uint4*>(in)[2 * t], b = reinterpret_cast<const uint4*>(in)[2 * t + 1];
    reinterpret_cast<uint4*>(out)[t] = make_uint4(a.x | (a.y << 16), a.z | (a.w << 16), b.x | (b.y << 16), b.z | (b.w << 16));
  }
  for (int64_t t = 8 * n8 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = (uint16_t)in[t];
}

// Host-format conversion: float64 / int64 residues <-> uint32 device storage.  The
// reference validates canonical residues when a DenseMatrix is built (field.py:140-147,
// ValueError); here the conversion flags any entry outside [0, p) (or a non-integral /
// NaN double) and stores 0 for it, and the caller raises PLUQ_EINVAL before factoring.
__global__ void from_f64_kernel(const double* in, uint32_t* out, int64_t count, uint32_t p, int* bad) {
  bool b = false;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x) {
    const double v = in[t];
    const bool ok = v >= 0.0 && v < (double)p && v == floor(v);
    out[t] = ok ? (uint32_t)v : 0u;
    b |= !ok;
  }
  if (bad && __syncthreads_or(b) && threadIdx.x == 0) atomicOr(bad, 1);
}
__global__ void to_f64_kernel(const uint32_t* in, double* out, int64_t count) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = (double)in[t];
}
__global__ void from_i64_kernel(const int64_t* in, uint32_t* out, int64_t count, uint32_t p, int* bad) {
  bool b = false;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = in[t];
    const bool ok = v >= 0 && v < (int64_t)p;
    out[t] = ok ? (uint32_t)v : 0u;
    b |= !ok;
  }
  if (bad && __syncthreads_or(b) && threadIdx.x == 0) atomicOr(bad, 1);
}
__global__ void to_i64_kernel(const uint32_t* in, int64_t* out, int64_t count) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = (int64_t)in[t];
}

// flag <- 1 if a device view holds an entry >= p (uint32 storage: a negative int32 tensor
// entry reads as >= 2^31 > p).  One read of the view, 16-byte loads when rows are aligned.
__global__ void range_check_kernel(View x, uint32_t p, int* flag) {
  bool bad = false;
  const bool vec = (x.ld % 4) == 0 && (reinterpret_cast<uintptr_t>(x.a) & 15) == 0;
  const int n4 = vec ? x.n / 4 : 0;
  for (int64_t i = blockIdx.y; i < x.m; i += gridDim.y) {
    const uint32_t* xr = x.row((int)i);
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n4; j += gridDim.x * blockDim.x) {
      const uint4 q = reinterpret_cast<const uint4*>(xr)[j];
      bad |= (q.x >= p) | (q.y >= p) | (q.z >= p) | (q.w >= p);
    }
    for (int j = 4 * n4 + blockIdx.x * blockDim.x + threadIdx.x; j < x.n; j += gridDim.x * blockDim.x) bad |= xr[j] >= p;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

}  // namespace pluq
