// Diagonal-block kernel of the speculative blocked LU (Driver::speculative_lu):
// unpivoted LU of one block of at most 128 x 128 in one CTA, register-resident with
// lazy reduction.  Same contract as diag_lazy_kernel (pluq_kernels.cuh): the block is
// factored in place; on a zero pivot at t the entries with i < t or j < t hold the
// factors of the first t pivots, the trailing block keeps its original values, and
// (status, stop) report (k0, t).
//
// Layout: 16 warps; warp w owns rows 8w..8w+7, lane l owns columns 4l..4l+3, every
// element a 64-bit accumulator taking one IMAD.WIDE per pivot step.  Step t publishes
// w_j = -U[t][j] / U[t][t] (owner warp of row t) and c_i = Schur[i][t] (each warp for
// its own rows, reduced by 8 lanes after a shared-memory transposition), so the update
// is acc[i][j] += c_i * w_j.  Per step and CTA barrier the critical chain is: column t+1
// updated first, the owner warp of row t+1 completes and reduces that row (4 values per
// lane, interleaved with its column reduction), inverts the pivot (shared-memory table
// when p < 2^16), scales and publishes; the remaining 24 products per thread follow.
// The t loop is unrolled by 8 so that the register row (t+1) % 8 and the register
// column (t+1) % 4 are compile-time constants (no dynamic register indexing, small code).
#pragma once
#include "pluq_common.cuh"

namespace pluq {

template <bool kSmall>
__device__ __forceinline__ uint32_t dg_red(unsigned long long x, const ModP& mp, uint32_t e32) {
  if (kSmall) {  // x < 2^40 (128 products of (p-1)^2 < 2^32 plus p): hi < 2^8
    const uint32_t lo = reduce32((uint32_t)x, mp);
    return reduce32(lo + (uint32_t)(x >> 32) * e32, mp);
  }
  return reduce64(x, mp);
}

template <bool kSmall>
__device__ __forceinline__ uint32_t dg_mul(uint32_t a, uint32_t b, const ModP& mp) {
  if (kSmall) return reduce32(a * b, mp);
  return reduce64((unsigned long long)a * b, mp);
}

inline size_t diag_reg_smem(bool tab) {
  return (size_t)128 * 132 * 4 + (tab ? 65536 * 2 : 0);
}

// kSmall: p < 2^16 with the inverse table (staged in shared memory); else requires
// 128 (p-1)^2 + p < 2^64 (mp.kchunk >= 130) and inverts with extended Euclid.
// kRev: warp w owns rows 8(15 - w).. instead of 8w..: the warp that owns the pivot row is then
// always the HIGHEST-numbered warp of its scheduler that still has active rows (finished rows
// belong to higher-numbered warps), and the warp arbiter favours the highest warp id — the
// pivot chain is no longer issued behind the other warps' bulk updates.
template <bool kSmall, bool kRev = true>
__global__ void __launch_bounds__(512, 1) diag_reg_kernel(View blk, ModP mp, const uint16_t* invtab, int* stop,
                                                           int* status, int k0) {
  if (stop && *reinterpret_cast<const volatile int*>(stop)) return;
  constexpr int B = 128, LDO = B + 4;
  extern __shared__ __align__(16) uint32_t smem_dyn[];
  __shared__ __align__(16) uint32_t s_c[2][B];
  __shared__ __align__(16) uint32_t s_w[2][B];
  __shared__ uint32_t s_inv[2];
  __shared__ __align__(16) unsigned long long s_tr[16][8];
  uint32_t* out = smem_dyn;                                               // [B][LDO]
  uint16_t* tab = reinterpret_cast<uint16_t*>(smem_dyn + B * LDO);        // [p] (kSmall)
  const int m = blk.m, n = blk.n, mn = min(m, n);
  const int tid = threadIdx.x, lane = tid & 31, w = kRev ? 15 - (tid >> 5) : (tid >> 5);  // logical warp
  const int r0 = 8 * w, j0 = 4 * lane;
  const uint32_t e32 = kSmall ? (uint32_t)((1ull << 32) % mp.p) : 0u;
  if (kSmall) {  // stage the inverse table with cp.async: every chunk in flight at once
    const int chunks = (int)((mp.p + 7) / 8);
    for (int q = tid; q < chunks; q += 512) {
      const unsigned sa = (unsigned)__cvta_generic_to_shared(tab + 8 * q);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(invtab + 8 * q));
    }
    asm volatile("cp.async.commit_group;\n" ::);
  }
  unsigned long long acc[8][4];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int i = r0 + r;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = j0 + q;
      const uint32_t v = (i < m && j < n) ? blk.at(i, j) : 0u;
      acc[r][q] = v;
      out[i * LDO + j] = v;
    }
  }
  if (kSmall) asm volatile("cp.async.wait_all;\n" ::);
  __syncthreads();  // table staged
  auto pinv = [&](uint32_t d) -> uint32_t { return d ? (kSmall ? (uint32_t)tab[d] : invmod(d, mp)) : 0u; };
  auto reload = [&](uint32_t (&c)[8], uint32_t (&wv)[4], int bb) {
    const uint4 ww = *reinterpret_cast<const uint4*>(&s_w[bb][j0]);
    wv[0] = ww.x; wv[1] = ww.y; wv[2] = ww.z; wv[3] = ww.w;
    const uint4 c0 = *reinterpret_cast<const uint4*>(&s_c[bb][r0]);
    const uint4 c1 = *reinterpret_cast<const uint4*>(&s_c[bb][r0 + 4]);
    c[0] = c0.x; c[1] = c0.y; c[2] = c0.z; c[3] = c0.w;
    c[4] = c1.x; c[5] = c1.y; c[6] = c1.z; c[7] = c1.w;
  };
  uint32_t my_c = 0;  // lanes < 8: L numerator of row r0 + lane for the current column
  if (w == 0 && mn > 0) {  // row 0 is final
    const uint32_t d = __shfl_sync(0xffffffffu, (uint32_t)acc[0][0], 0);
    const uint32_t iv = pinv(d);
    uint32_t wv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t u = (uint32_t)acc[0][q];
      wv[q] = (j0 + q > 0 && u) ? dg_mul<kSmall>(mp.p - u, iv, mp) : 0u;
    }
    *reinterpret_cast<uint4*>(&s_w[0][j0]) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
    if (lane == 0) s_inv[0] = iv;
  }
  if (lane == 0) {
#pragma unroll
    for (int r = 0; r < 8; ++r) s_tr[w][r] = acc[r][0];
  }
  __syncwarp();
  if (lane < 8) {
    my_c = (uint32_t)s_tr[w][lane];
    s_c[0][r0 + lane] = r0 + lane > 0 ? my_c : 0u;
  }
  int stop_t = mn;
  for (int tb = 0; tb < mn; tb += 8) {
#pragma unroll
    for (int tr = 0; tr < 8; ++tr) {
      const int t = tb + tr;
      if (t >= mn) break;  // block-uniform
      const int bb = tr & 1, nb = bb ^ 1;
      const int Q1 = (tr + 1) & 3;  // register column of t+1 in its owner lane
      const int RR = (tr + 1) & 7;  // register row of t+1 in its owner warp
      __syncthreads();  // operands of step t published
      const uint32_t iv = s_inv[bb];
      if (iv == 0u) { stop_t = t; break; }
      const int t1 = t + 1, l1 = t1 >> 2;
      const bool more = t1 < mn;
      const bool active = r0 + 7 > t;
      const bool colact = more && r0 + 7 > t1;
      const bool piv = more && w == (t1 >> 3);
      if (lane < 8 && r0 + lane > t && r0 + lane < m) out[(r0 + lane) * LDO + t] = dg_mul<kSmall>(my_c, iv, mp);
      uint32_t c[8], wv[4] = {0u, 0u, 0u, 0u};
      if (active) {
        reload(c, wv, bb);
#pragma unroll
        for (int r = 0; r < 8; ++r) acc[r][Q1] += (unsigned long long)c[r] * wv[Q1];
      } else {
#pragma unroll
        for (int r = 0; r < 8; ++r) c[r] = 0u;
      }
      if (colact) {
        if (lane == l1) {
#pragma unroll
          for (int r = 0; r < 8; ++r) s_tr[w][r] = acc[r][Q1];
        }
        __syncwarp();
      }
      if (piv) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (q != Q1) acc[RR][q] += (unsigned long long)c[RR] * wv[q];  // row t+1 complete
        const unsigned long long xc = s_tr[w][lane & 7];
        uint32_t u[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) u[q] = dg_red<kSmall>(acc[RR][q], mp, e32);
        const uint32_t cvr = dg_red<kSmall>(xc, mp, e32);
        const uint32_t d = __shfl_sync(0xffffffffu, u[Q1], l1);
        const uint32_t ivn = pinv(d);
        uint32_t wn[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int j = j0 + q;
          wn[q] = (j > t1 && u[q]) ? dg_mul<kSmall>(mp.p - u[q], ivn, mp) : 0u;
          if (d != 0u && j >= t1 && j < n) out[t1 * LDO + j] = u[q];  // U row (original kept on a zero pivot)
        }
        *reinterpret_cast<uint4*>(&s_w[nb][j0]) = make_uint4(wn[0], wn[1], wn[2], wn[3]);
        if (lane == 0) s_inv[nb] = ivn;
        if (colact && lane < 8) {
          my_c = cvr;
          s_c[nb][r0 + lane] = r0 + lane > t1 ? cvr : 0u;
        }
        reload(c, wv, bb);  // short live ranges: operands re-read from shared memory
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (q != Q1 && r != RR) acc[r][q] += (unsigned long long)c[r] * wv[q];
      } else {
        if (colact && lane < 8) {
          my_c = dg_red<kSmall>(s_tr[w][lane], mp, e32);
          s_c[nb][r0 + lane] = r0 + lane > t1 ? my_c : 0u;
        }
        if (active) {
          reload(c, wv, bb);
#pragma unroll
          for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (q != Q1) acc[r][q] += (unsigned long long)c[r] * wv[q];
        }
      }
    }
    if (stop_t < mn) break;
  }
  __syncthreads();
  for (int idx = tid; idx < m * n; idx += 512) {
    const int i = idx / n, j = idx - (idx / n) * n;
    blk.at(i, j) = out[i * LDO + j];
  }
  if (tid == 0 && stop_t < mn) {
    status[0] = k0;
    status[1] = stop_t;
    __threadfence();
    atomicExch(stop, 1);
  }
}

}  // namespace pluq
