// Diagonal-block kernel of the speculative blocked LU, run-ahead version (same contract as
// diag_reg_kernel, pluq_diag.cuh): unpivoted LU of one block of at most 128 x 128 in one CTA;
// on a zero pivot at t the entries with i < t or j < t hold the factors of the first t
// pivots, the trailing block keeps its original values, and (status, stop) report (k0, t).
//
// diag_reg_kernel runs its 128 pivot steps in lock-step: one CTA barrier per step, and every
// step waits for the warp that owns the pivot row to reduce it, invert the pivot and publish
// the scaled row (~0.9 us per step, 114 us per block, issue slots 25 % busy).  Here the steps
// are decoupled:
//  * warp g owns rows 8g..8g+7 (lane = 4 columns, 64-bit lazy accumulators) and is the
//    PRODUCER of the pivot rows t = 8g..8g+7: all it needs for them is in its own registers
//    (its rows, its own column values, the w rows it produced itself), so it runs its eight
//    pivots back to back without waiting for anybody;
//  * every produced row w_t = -U[t][:] / U[t][t] goes to its own slot of a 128-slot ring in
//    shared memory and is announced on its own single-use mbarrier; the other warps consume
//    the slots in order at their own pace (acc[i][j] += c_i w_j, c_i their own column value)
//    and do the transposition / reduction of their next column BEFORE they wait;
//  * factors are written straight to global memory as they become final (U row by its
//    producer, L column entries by the row owners), so a zero pivot leaves the trailing block
//    untouched without a staging copy, and finished warps simply exit;
//  * with one warp on the critical path the cost of a pivot is that warp's INSTRUCTION count
//    (a lone warp issues a dependent instruction every ~4-5 cycles), so for 512 <= p < 2^16
//    (kFast) the reductions are 5 instructions each: x < 2^39 reduces with one Barrett
//    quotient taken from x >> 8 (short by at most 1, see red40), products of residues with
//    the 32-bit Barrett quotient (short by at most 1); the producer's own L-column entries
//    are scaled and stored after its eight pivots;
//  * logical warp g is hardware warp 15 - g: the producer is then the highest-numbered warp
//    of its scheduler that still has work, which the warp arbiter favours.
#pragma once
#include "pluq_diag.cuh"

namespace pluq {

#ifdef PLUQ_DIAG_TRACE  // microbenchmark only: publication time of every pivot, consumption time in the last warp
__device__ long long g_diag_trace[256];
#endif

inline size_t diag_run_smem(bool tab) { return (size_t)128 * 128 * 4 + (tab ? 65536 * 2 : 0); }

__device__ __forceinline__ uint32_t dr_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void dr_mbar_wait(uint64_t* bar) {  // single-use barrier: phase 0
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(dr_smem_u32(bar))
      : "memory");
}

// x mod p for x < 2^39 and 512 <= p < 2^16: q = floor((x >> 8) mu40 / 2^32), mu40 = floor(2^40 / p),
// satisfies x/p - 1 < q <= x/p (the truncations lose less than x/2^40 + 2^8/p < 1), so one
// conditional subtraction finishes; the remainder x - q p < 2p fits 32-bit wrap-around arithmetic.
__device__ __forceinline__ uint32_t red40(unsigned long long x, uint32_t p, uint32_t np, uint32_t mu40) {
  const uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
  const uint32_t q = __umulhi(__funnelshift_r(lo, hi, 8), mu40);
  const uint32_t r = q * np + lo;  // np = -p mod 2^32: one IMAD
  return min(r, r - p);
}
// a b mod p for a, b <= p < 2^16 (a b < 2^32): mu32 = floor((2^32 - 1) / p), quotient short by at most 1.
__device__ __forceinline__ uint32_t mul16(uint32_t a, uint32_t b, uint32_t p, uint32_t np, uint32_t mu32) {
  const uint32_t x = a * b;
  const uint32_t r = __umulhi(x, mu32) * np + x;
  return min(r, r - p);
}

// kFull: the block is exactly 128 x 128 with 16-byte aligned rows (no per-step bounds checks, whole
// 16-byte stores of the U row pieces); the driver uses the kernel only then.
template <bool kSmall, bool kFast, bool kFull = false>
__global__ void __launch_bounds__(512, 1) diag_run_kernel(View blk, ModP mp, const uint16_t* invtab, int* stop,
                                                           int* status, int k0) {
  if (stop && *reinterpret_cast<const volatile int*>(stop)) return;
  constexpr int B = 128;
  extern __shared__ __align__(16) uint32_t smem_dyn[];
  __shared__ __align__(8) uint64_t s_full[B];
  __shared__ uint32_t s_inv[B];
  __shared__ __align__(16) unsigned long long s_tr[16][8];
  __shared__ __align__(16) uint32_t s_cw[16][8];
  uint32_t* ring = smem_dyn;                                         // [B][B] scaled pivot rows
  uint16_t* tab = reinterpret_cast<uint16_t*>(smem_dyn + B * B);     // [p] (kSmall)
  const int m = kFull ? 128 : blk.m, n = kFull ? 128 : blk.n, mn = min(m, n);
  const int tid = threadIdx.x, lane = tid & 31, pw = tid >> 5, g = 15 - pw;
  const int r0 = 8 * g, j0 = 4 * lane;
  const uint32_t P = mp.p, NP = 0u - mp.p;
  const uint32_t e32 = kSmall ? (uint32_t)((1ull << 32) % P) : 0u;
  const uint32_t mu40 = kFast ? (uint32_t)((1ull << 40) / P) : 0u;
  const uint32_t mu32 = mp.mu32;
  auto red = [=](unsigned long long x) -> uint32_t { return kFast ? red40(x, P, NP, mu40) : dg_red<kSmall>(x, mp, e32); };
  auto mul = [=](uint32_t a, uint32_t b) -> uint32_t { return kFast ? mul16(a, b, P, NP, mu32) : dg_mul<kSmall>(a, b, mp); };
  if (kSmall) {
    const int chunks = (int)((P + 7) / 8);
    for (int q = tid; q < chunks; q += 512) {
      const unsigned sa = (unsigned)__cvta_generic_to_shared(tab + 8 * q);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(invtab + 8 * q));
    }
    asm volatile("cp.async.commit_group;\n" ::);
  }
  if (tid < B) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(dr_smem_u32(&s_full[tid])));
  unsigned long long acc[8][4];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int i = r0 + r;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = j0 + q;
      acc[r][q] = (i < m && j < n) ? blk.at(i, j) : 0u;
    }
  }
  if (kSmall) asm volatile("cp.async.wait_all;\n" ::);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();  // table staged (tab[0] = 0), barriers initialised; no CTA-wide barrier after this one
  auto pinv = [&](uint32_t d) -> uint32_t { return kSmall ? (uint32_t)tab[d] : (d ? invmod(d, mp) : 0u); };
  const int ci = r0 + (lane & 7);                       // row whose column value this lane reduces
  uint32_t* lcol = blk.a + (int64_t)ci * blk.ld;        // its row in global memory (L entries)
  // whole 16-byte stores of U row pieces: full-width block, rows and base 16-byte aligned
  const bool uvec = kFull || (n == B && (blk.ld & 3) == 0 && (reinterpret_cast<uintptr_t>(blk.a) & 15) == 0);
  bool stopped = false;
  for (int tb = 0; tb < mn && !stopped; tb += 8) {
    if (r0 + 7 < tb) break;  // every row of this warp is final
    if ((tb >> 3) == g) {
      // ---- producer of the pivots tb .. tb + 7: no waits inside ----
      uint32_t lc[8], li[8];  // this lane's column value and the pivot inverse per step (L entries, stored below)
      uint32_t* ubase = blk.a + (int64_t)tb * blk.ld + j0;
      int done = 0;
#pragma unroll
      for (int tr = 0; tr < 8; ++tr) {
        const int t = tb + tr;
        if (!kFull && t >= mn) break;
        const int lt = t >> 2, Q = tr & 3;
        if (lane == lt) {
#pragma unroll
          for (int r = 0; r < 8; ++r)
            if (r > tr) s_tr[pw][r] = acc[r][Q];
        }
        uint32_t u[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) u[q] = red(acc[tr][q]);  // row t is final
        // column value of the NEXT pivot row (row t + 1, held by lane lt): reduced and broadcast
        // by shuffle, off the shared-memory transposition, so that row t + 1 is complete right
        // after w_t is known — the pivot-to-pivot chain is red, shfl, table, mul, 4 IMADs
        uint32_t cf = 0u;
        if (tr < 7) cf = __shfl_sync(0xffffffffu, red(acc[tr < 7 ? tr + 1 : tr][Q]), lt);
        __syncwarp();
        const uint32_t cval = red(s_tr[pw][lane & 7]);
        if (lane < 8) s_cw[pw][lane] = ci > t ? cval : 0u;
        const uint32_t d = __shfl_sync(0xffffffffu, u[Q], lt);
        const uint32_t iv = pinv(d);
        const uint32_t niv = P - iv;
        uint32_t wv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) wv[q] = mul(u[q], niv);  // -U[t][j] / U[t][t], four independent chains
#pragma unroll
        for (int q = 0; q < 4; ++q) wv[q] = j0 + q > t ? wv[q] : 0u;
        *reinterpret_cast<uint4*>(&ring[t * B + j0]) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        if (lane == 0) s_inv[t] = iv;
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(dr_smem_u32(&s_full[t])) : "memory");
#ifdef PLUQ_DIAG_TRACE
        if (lane == 0) g_diag_trace[t] = clock64();
#endif
        if (__any_sync(0xffffffffu, iv == 0u)) {
          if (lane == 0) {
            status[0] = k0;
            status[1] = t;
            __threadfence();
            atomicExch(stop, 1);
          }
          stopped = true;
          break;
        }
        if (tr < 7) {
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[tr < 7 ? tr + 1 : tr][q] += (unsigned long long)cf * wv[q];  // row t + 1 complete
        }
        lc[tr] = cval;
        li[tr] = iv;
        done = tr + 1;
        {
          uint32_t* urow = ubase + (int64_t)tr * blk.ld;  // U row (original kept on a zero pivot)
          if (uvec) {  // lanes right of the pivot's lane: 16 bytes; the pivot's lane: its entries from Q on
            if (lane > lt) *reinterpret_cast<uint4*>(urow) = make_uint4(u[0], u[1], u[2], u[3]);
            if (lane == lt) {
#pragma unroll
              for (int q = 0; q < 4; ++q)
                if (q >= Q) urow[q] = u[q];
            }
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (j0 + q >= t && j0 + q < n) urow[q] = u[q];
          }
        }
        if (tr < 6) {
          const uint4 c0 = *reinterpret_cast<const uint4*>(&s_cw[pw][0]);
          const uint4 c1 = *reinterpret_cast<const uint4*>(&s_cw[pw][4]);
          const uint32_t c[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
          const int Qn = (tr + 1) & 3;  // the next pivot column first: its transposition starts the next step
#pragma unroll
          for (int r = 0; r < 8; ++r)
            if (r > tr + 1) acc[r][Qn] += (unsigned long long)c[r] * wv[Qn];
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            if (r <= tr + 1) continue;  // rows up to t are final, row t + 1 is done above
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (q != Qn) acc[r][q] += (unsigned long long)c[r] * wv[q];
          }
        }
      }
      // L entries of this warp's rows in the columns it produced
      if (lane < 8 && ci < m) {
#pragma unroll
        for (int tr = 0; tr < 8; ++tr)
          if (tr < done && ci > tb + tr) lcol[tb + tr] = mul(lc[tr], li[tr]);
      }
      break;  // every row of this warp is final
    }
    // ---- consumer of the pivots tb .. tb + 7 ----
    // Column t of this warp's rows is final after step t - 1: it is transposed through shared
    // memory (lane t / 4 holds it; 8 lanes reduce one value each) BEFORE the wait for w_t, and
    // the next column is updated first so that its transposition overlaps the rest of the
    // update.  The L entries c_i / U[t][t] are scaled and stored after the eight steps.
    uint32_t lc[8], li[8];
    int done = 0;
    auto transpose_out = [&](int Q, int lt) {
      if (lane == lt) {
#pragma unroll
        for (int r = 0; r < 8; r += 2)
          *reinterpret_cast<ulonglong2*>(&s_tr[pw][r]) = make_ulonglong2(acc[r][Q], acc[r + 1][Q]);
      }
    };
    transpose_out(0, tb >> 2);
#pragma unroll
    for (int tr = 0; tr < 8; ++tr) {
      const int t = tb + tr;
      if (!kFull && t >= mn) break;
      const int Q = tr & 3, Qn = (tr + 1) & 3;
      __syncwarp();
      const uint32_t cval = red(s_tr[pw][lane & 7]);
      if (lane < 8) s_cw[pw][lane] = cval;
      __syncwarp();
      const uint4 c0 = *reinterpret_cast<const uint4*>(&s_cw[pw][0]);
      const uint4 c1 = *reinterpret_cast<const uint4*>(&s_cw[pw][4]);
      const uint32_t c[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
      dr_mbar_wait(&s_full[t]);
      const uint4 ww = *reinterpret_cast<const uint4*>(&ring[t * B + j0]);
      const uint32_t iv = s_inv[t];
      if (__any_sync(0xffffffffu, iv == 0u)) { stopped = true; break; }
      lc[tr] = cval;
      li[tr] = iv;
      done = tr + 1;
      const uint32_t wv[4] = {ww.x, ww.y, ww.z, ww.w};
      (void)Q;
#pragma unroll
      for (int r = 0; r < 8; ++r) acc[r][Qn] += (unsigned long long)c[r] * wv[Qn];
      if (tr < 7) transpose_out(Qn, (t + 1) >> 2);  // column t + 1 is final: start its transposition
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (q != Qn) acc[r][q] += (unsigned long long)c[r] * wv[q];
#ifdef PLUQ_DIAG_TRACE
      if (lane == 0 && g == 15) g_diag_trace[128 + t] = clock64();
#endif
    }
    if (lane < 8 && ci < m) {
#pragma unroll
      for (int tr = 0; tr < 8; ++tr)
        if (tr < done) lcol[tb + tr] = mul(lc[tr], li[tr]);  // L column entries
    }
  }
}

}  // namespace pluq
