// Global-memory kernels used by the host recursion driver and the C ABI.
#pragma once
#include "pluq_small.cuh"

namespace pluq {

// ---------------------------------------------------------------------------------
// Small-node / batched PLUQ: one CTA per block, block staged through shared memory.
// ---------------------------------------------------------------------------------
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
};

__global__ void small_pluq_kernel(SmallArgs args) {
  extern __shared__ __align__(16) uint32_t smem_dyn[];
  __shared__ BcShared sh;
  __shared__ Counts cnt;
  const int m = args.m, n = args.n;
  const int lds = n | 1;
  uint32_t* ga = args.a + (int64_t)blockIdx.x * args.bstride;
  uint32_t* sa = smem_dyn;
  int* stk = reinterpret_cast<int*>(sa + (((int64_t)m * lds + 3) & ~3ll));
  for (int idx = threadIdx.x; idx < m * n; idx += blockDim.x) {
    int i = idx / n, j = idx - i * n;
    sa[i * lds + j] = ga[(int64_t)i * args.lda + j];
  }
  if (threadIdx.x == 0) { cnt.mul = cnt.add = cnt.inv = cnt.red = 0; }
  __syncthreads();
  SmallCtx c{args.mp, args.threshold, &cnt, &sh};
  View x{sa, lds, m, n};
  int* P = stk; int* Q = P + m; int* top = Q + n;
  const int r = rec_smem(x, P, Q, top, c);
  for (int idx = threadIdx.x; idx < m * n; idx += blockDim.x) {
    int i = idx / n, j = idx - i * n;
    ga[(int64_t)i * args.lda + j] = sa[i * lds + j];
  }
  int* po = args.p_out + (int64_t)blockIdx.x * m;
  int* qo = args.q_out + (int64_t)blockIdx.x * n;
  for (int t = threadIdx.x; t < m; t += blockDim.x) po[t] = P[t];
  for (int t = threadIdx.x; t < n; t += blockDim.x) qo[t] = Q[t];
  if (threadIdx.x == 0) {
    args.r_out[blockIdx.x] = r;
    unsigned long long* co = args.cnt_out + (args.cnt_accumulate ? 0 : 4 * (int64_t)blockIdx.x);
    if (args.cnt_accumulate) {
      atomicAdd(co + 0, cnt.mul); atomicAdd(co + 1, cnt.add);
      atomicAdd(co + 2, cnt.inv); atomicAdd(co + 3, cnt.red);
    } else {
      co[0] = cnt.mul; co[1] = cnt.add; co[2] = cnt.inv; co[3] = cnt.red;
    }
  }
}

// Dynamic shared memory of small_pluq_kernel: block (odd pitch) + P/Q + recursion stack.
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
__global__ void __launch_bounds__(256) simt_gemm_kernel(View c, View a, View b, ModP mp) {
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
    for (int idx = tid; idx < SG_BM * SG_BK; idx += 256) {
      int i = idx / SG_BK, kk = idx % SG_BK;
      int gi = m0 + i, gk = k0 + kk;
      As[kk][i] = (gi < m && gk < k) ? a.at(gi, gk) : 0u;
    }
    for (int idx = tid; idx < SG_BK * SG_BN; idx += 256) {
      int kk = idx / SG_BN, j = idx % SG_BN;
      int gk = k0 + kk, gj = n0 + j;
      Bs[kk][j] = (gk < k && gj < n) ? b.at(gk, gj) : 0u;
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
// TRSM base kernels (r <= 64): L / U resident in shared memory.
// ---------------------------------------------------------------------------------
constexpr int TR_BASE = 64;

// B <- L^-1 B for a strip of 128 columns per CTA (thread per column).
__global__ void __launch_bounds__(128) trsm_llu_base_kernel(View l, View b, ModP mp) {
  __shared__ uint32_t Ls[TR_BASE][TR_BASE];
  __shared__ uint32_t Bs[TR_BASE][128];
  const int r = l.m, n = b.n;
  const int c0 = blockIdx.x * 128;
  for (int idx = threadIdx.x; idx < r * r; idx += 128) {
    int i = idx / r, j = idx % r;
    Ls[i][j] = l.at(i, j);
  }
  for (int i = 0; i < r; ++i) {
    int c = c0 + threadIdx.x;
    Bs[i][threadIdx.x] = c < n ? b.at(i, c) : 0u;
  }
  __syncthreads();
  const int c = threadIdx.x;
  const bool fast = (uint64_t)r <= mp.kchunk;
  for (int i = 1; i < r; ++i) {
    uint64_t acc = 0, cntk = 0;
    for (int t = 0; t < i; ++t) {
      acc += (uint64_t)Ls[i][t] * Bs[t][c];
      if (!fast && ++cntk == mp.kchunk) { acc = reduce64(acc, mp); cntk = 0; }
    }
    Bs[i][c] = submod(Bs[i][c], reduce64(acc, mp), mp);
  }
  __syncthreads();
  for (int i = 0; i < r; ++i) {
    int cc = c0 + threadIdx.x;
    if (cc < n) b.at(i, cc) = Bs[i][threadIdx.x];
  }
}

// B <- B U^-1 for a strip of 64 rows per CTA (thread per row, 64 threads).
__global__ void __launch_bounds__(64) trsm_ru_base_kernel(View b, View u, ModP mp) {
  __shared__ uint32_t Us[TR_BASE][TR_BASE + 1];
  __shared__ uint32_t Bs[64][TR_BASE + 1];
  __shared__ uint32_t inv[TR_BASE];
  const int m = b.m, r = u.m;
  const int r0 = blockIdx.x * 64;
  for (int idx = threadIdx.x; idx < r * r; idx += 64) {
    int i = idx / r, j = idx % r;
    Us[i][j] = u.at(i, j);
  }
  for (int j = threadIdx.x; j < r; j += 64) inv[j] = invmod(u.at(j, j), mp);
  for (int idx = threadIdx.x; idx < 64 * r; idx += 64) {
    int i = idx / r, j = idx % r;
    Bs[i][j] = (r0 + i < m) ? b.at(r0 + i, j) : 0u;
  }
  __syncthreads();
  const int i = threadIdx.x;
  const bool fast = (uint64_t)r <= mp.kchunk;
  for (int j = 0; j < r; ++j) {
    uint64_t acc = 0, cntk = 0;
    for (int t = 0; t < j; ++t) {
      acc += (uint64_t)Bs[i][t] * Us[t][j];
      if (!fast && ++cntk == mp.kchunk) { acc = reduce64(acc, mp); cntk = 0; }
    }
    Bs[i][j] = mulmod(submod(Bs[i][j], reduce64(acc, mp), mp), inv[j], mp);
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < 64 * r; idx += 64) {
    int ii = idx / r, j = idx % r;
    if (r0 + ii < m) b.at(r0 + ii, j) = Bs[ii][j];
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
__global__ void rows_to_tmp_kernel(View x, const int* src, int nmv, uint32_t* tmp) {
  for (int q = blockIdx.y; q < nmv; q += gridDim.y) {
    const uint32_t* sr = x.row(src[q]);
    uint32_t* tr = tmp + (int64_t)q * x.n;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < x.n; j += gridDim.x * blockDim.x) tr[j] = sr[j];
  }
}
__global__ void tmp_to_rows_kernel(View x, const int* dst, int nmv, const uint32_t* tmp) {
  for (int q = blockIdx.y; q < nmv; q += gridDim.y) {
    uint32_t* dr = x.row(dst[q]);
    const uint32_t* tr = tmp + (int64_t)q * x.n;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < x.n; j += gridDim.x * blockDim.x) dr[j] = tr[j];
  }
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

// flag <- 1 if the block holds any nonzero (zero-block short-circuit).
__global__ void nonzero_kernel(View x, int* flag) {
  bool nz = false;
  for (int i = blockIdx.y; i < x.m; i += gridDim.y) {
    const uint32_t* xr = x.row(i);
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < x.n; j += gridDim.x * blockDim.x) nz |= xr[j] != 0u;
  }
  if (__syncthreads_or(nz) && threadIdx.x == 0) atomicOr(flag, 1);
}

__global__ void copy_view_kernel(View dst, View src) {
  for (int i = blockIdx.y; i < dst.m; i += gridDim.y)
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < dst.n; j += gridDim.x * blockDim.x)
      dst.at(i, j) = src.at(i, j);
}

// Host-format conversion: float64 / int64 residues <-> uint32 device storage.
__global__ void from_f64_kernel(const double* in, uint32_t* out, int64_t count) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = (uint32_t)in[t];
}
__global__ void to_f64_kernel(const uint32_t* in, double* out, int64_t count) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = (double)in[t];
}
__global__ void from_i64_kernel(const int64_t* in, uint32_t* out, int64_t count) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = (uint32_t)in[t];
}
__global__ void to_i64_kernel(const uint32_t* in, int64_t* out, int64_t count) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = (int64_t)in[t];
}

}  // namespace pluq
