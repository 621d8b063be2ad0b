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
  const uint16_t* invtab;       // inverse table when p < 2^16 (else nullptr)
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
  SmallCtx c{args.mp, args.threshold, &cnt, &sh, args.invtab};
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

// out[b] = inverse of the b-th 64x64 diagonal block of U (upper, nonzero diagonal); 64 threads.
__global__ void __launch_bounds__(64) trinv_upper_kernel(View u, uint32_t* out, ModP mp, const uint16_t* invtab) {
  __shared__ uint32_t Us[TR_BASE][TR_BASE + 1];
  __shared__ uint32_t X[TR_BASE][TR_BASE + 1];
  __shared__ uint32_t dinv[TR_BASE];
  const int base = blockIdx.x * TR_BASE;
  const int w = min(TR_BASE, u.m - base);
  for (int idx = threadIdx.x; idx < w * w; idx += 64) {
    int i = idx / w, j = idx % w;
    Us[i][j] = u.at(base + i, base + j);
  }
  __syncthreads();
  if ((int)threadIdx.x < w) dinv[threadIdx.x] = invtab ? invtab[Us[threadIdx.x][threadIdx.x]] : invmod(Us[threadIdx.x][threadIdx.x], mp);
  __syncthreads();
  const int j = threadIdx.x;
  if (j < w) {
    for (int i = 0; i < w; ++i) X[i][j] = 0;
    X[j][j] = dinv[j];
    for (int i = j - 1; i >= 0; --i) {
      uint32_t s = acc_dot(&Us[i][i + 1], 1, &X[i + 1][j], TR_BASE + 1, j - i, mp);
      X[i][j] = mulmod(s ? mp.p - s : 0u, dinv[i], mp);
    }
  }
  __syncthreads();
  uint32_t* o = out + (size_t)blockIdx.x * TR_BASE * TR_BASE;
  for (int idx = threadIdx.x; idx < w * w; idx += 64) o[(idx / w) * TR_BASE + idx % w] = X[idx / w][idx % w];
}

// out[b] = inverse of the b-th diagonal block of unit-lower L (diagonal implicit 1); 64 threads.
__global__ void __launch_bounds__(64) trinv_lower_unit_kernel(View l, uint32_t* out, ModP mp) {
  __shared__ uint32_t Ls[TR_BASE][TR_BASE + 1];
  __shared__ uint32_t X[TR_BASE][TR_BASE + 1];
  const int base = blockIdx.x * TR_BASE;
  const int w = min(TR_BASE, l.m - base);
  for (int idx = threadIdx.x; idx < w * w; idx += 64) {
    int i = idx / w, j = idx % w;
    Ls[i][j] = l.at(base + i, base + j);
  }
  __syncthreads();
  const int j = threadIdx.x;
  if (j < w) {
    for (int i = 0; i < w; ++i) X[i][j] = 0;
    X[j][j] = 1;
    for (int i = j + 1; i < w; ++i) {
      uint32_t s = acc_dot(&Ls[i][j], 1, &X[j][j], TR_BASE + 1, i - j, mp);
      X[i][j] = s ? mp.p - s : 0u;
    }
  }
  __syncthreads();
  uint32_t* o = out + (size_t)blockIdx.x * TR_BASE * TR_BASE;
  for (int idx = threadIdx.x; idx < w * w; idx += 64) o[(idx / w) * TR_BASE + idx % w] = X[idx / w][idx % w];
}

// B <- B * Uinv for a w-column block (w <= 64): one CTA owns 64 rows of B (in place).
__global__ void __launch_bounds__(256) trsm_apply_right_kernel(View b, const uint32_t* uinv, ModP mp) {
  __shared__ uint32_t Bs[64][TR_BASE + 1];
  __shared__ uint32_t Ui[TR_BASE][TR_BASE + 1];
  const int w = b.n, r0 = blockIdx.x * 64, rows = min(64, b.m - r0);
  for (int idx = threadIdx.x; idx < w * w; idx += 256) Ui[idx / w][idx % w] = uinv[(idx / w) * TR_BASE + idx % w];
  for (int idx = threadIdx.x; idx < rows * w; idx += 256) Bs[idx / w][idx % w] = b.at(r0 + idx / w, idx % w);
  __syncthreads();
  const int rr = threadIdx.x >> 2, c0 = (threadIdx.x & 3) * 16;
  uint32_t res[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int cc = c0 + q;
    // X[rr][cc] = sum_{t<=cc} B[rr][t] Uinv[t][cc]
    res[q] = (rr < rows && cc < w) ? acc_dot(&Bs[rr][0], 1, &Ui[0][cc], TR_BASE + 1, cc + 1, mp) : 0u;
  }
  __syncthreads();
  if (rr < rows)
#pragma unroll
    for (int q = 0; q < 16; ++q)
      if (c0 + q < w) b.at(r0 + rr, c0 + q) = res[q];
}

// B <- Linv * B for a w-row block (w <= 64): one CTA owns 64 columns of B (in place).
__global__ void __launch_bounds__(256) trsm_apply_left_kernel(const uint32_t* linv, View b, ModP mp) {
  __shared__ uint32_t Bs[TR_BASE][64 + 1];
  __shared__ uint32_t Li[TR_BASE][TR_BASE + 1];
  const int w = b.m, c0 = blockIdx.x * 64, cols = min(64, b.n - c0);
  for (int idx = threadIdx.x; idx < w * w; idx += 256) Li[idx / w][idx % w] = linv[(idx / w) * TR_BASE + idx % w];
  for (int idx = threadIdx.x; idx < w * 64; idx += 256) {
    int i = idx / 64, j = idx % 64;
    Bs[i][j] = j < cols ? b.at(i, c0 + j) : 0u;
  }
  __syncthreads();
  const int cc = threadIdx.x & 63, r0 = (threadIdx.x >> 6) * 16;
  uint32_t res[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int rr = r0 + q;
    // X[rr][cc] = sum_{t<=rr} Linv[rr][t] B[t][cc]
    res[q] = (rr < w && cc < cols) ? acc_dot(&Li[rr][0], 1, &Bs[0][cc], 65, rr + 1, mp) : 0u;
  }
  __syncthreads();
  if (cc < cols)
#pragma unroll
    for (int q = 0; q < 16; ++q)
      if (r0 + q < w) b.at(r0 + q, c0 + cc) = res[q];
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

// Table of inverses mod p (p < 2^16): tab[a] = a^-1, tab[0] = 0.
__global__ void invtab_kernel(uint16_t* tab, ModP mp) {
  for (uint32_t a = blockIdx.x * blockDim.x + threadIdx.x; a < mp.p; a += gridDim.x * blockDim.x)
    tab[a] = a ? (uint16_t)invmod(a, mp) : 0;
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
