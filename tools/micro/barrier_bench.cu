// Microbenchmark: cycles per step of typical per-pivot step patterns in one CTA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o barrier_bench barrier_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_bar(int iters, long long* out) {  // bare barrier
  __shared__ int s[1024];
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  if (threadIdx.x == 0) out[0] = (clock64() - t0) / iters;
  s[threadIdx.x] = 0;
}
__global__ void k_bar_smem(int iters, long long* out) {  // barrier + owner writes a row, all read it
  __shared__ uint32_t row[2][128];
  uint32_t acc = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if ((threadIdx.x >> 5) == (i & 15) && (threadIdx.x & 31) < 32) {
      row[i & 1][threadIdx.x & 31] = acc; row[i & 1][(threadIdx.x & 31) + 32] = acc + 1;
    }
    __syncthreads();
    acc += row[i & 1][(threadIdx.x + i) & 63];
  }
  if (threadIdx.x == 0) out[1] = (clock64() - t0) / iters;
  if (acc == 12345) out[5] = acc;
}
__global__ void k_bar_shfl_tab(int iters, long long* out, const uint16_t* tab) {  // barrier + shfl + global table
  __shared__ uint32_t piv[2];
  uint32_t acc = threadIdx.x + 1;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x == 0) piv[i & 1] = tab[(acc + i) & 0xffff];
    __syncthreads();
    acc = __shfl_sync(0xffffffffu, acc + piv[i & 1], (i & 31));
  }
  if (threadIdx.x == 0) out[2] = (clock64() - t0) / iters;
  if (acc == 12345) out[5] = acc;
}
__device__ __forceinline__ uint32_t red64(uint64_t x, uint64_t mu, uint32_t p) {
  uint64_t q = __umul64hi(x, mu);
  uint64_t r = x - q * p;
  r = r >= p ? r - p : r;
  r = r >= p ? r - p : r;
  return (uint32_t)r;
}
__global__ void k_bar_math(int iters, long long* out, uint32_t p) {  // barrier + 8 dependent mulmods
  uint64_t mu = ~0ull / p;
  uint32_t a = threadIdx.x + 3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 8; ++j) a = red64((uint64_t)a * (a + j), mu, p);
  }
  if (threadIdx.x == 0) out[3] = (clock64() - t0) / iters;
  if (a == 12345) out[5] = a;
}
__device__ __forceinline__ uint32_t red32(uint32_t x, uint32_t mu32, uint32_t p) {
  uint32_t q = __umulhi(x, mu32);
  uint32_t r = x - q * p;
  r = r >= p ? r - p : r;
  r = r >= p ? r - p : r;
  return r;
}
// x < 2^48, p < 2^16: x = hi*2^32 + lo, x mod p = (lo mod p + (hi*R mod p)) mod p, R = 2^32 mod p
__device__ __forceinline__ uint32_t red48(uint64_t x, uint32_t mu32, uint32_t R, uint32_t p) {
  const uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
  uint32_t t = red32(lo, mu32, p) + red32(hi * R, mu32, p);
  return t >= p ? t - p : t;
}
__global__ void k_bar_math32(int iters, long long* out, uint32_t p) {  // barrier + 8 dependent 32-bit reductions
  const uint32_t mu32 = 0xffffffffu / p, R = (uint32_t)((1ull << 32) % p);
  uint32_t a = threadIdx.x + 3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 8; ++j) a = red48((uint64_t)a * (a + j) * 37u, mu32, R, p);
  }
  if (threadIdx.x == 0) out[4] = (clock64() - t0) / iters;
  if (a == 12345) out[5] = a;
}
// FP64 reduction: x exact integer < 2^53, p < 2^16
__device__ __forceinline__ double redf(double x, double p, double pinv) {
  double q = floor(x * pinv);
  double r = fma(-q, p, x);
  r = r < 0.0 ? r + p : r;
  r = r >= p ? r - p : r;
  return r;
}
__global__ void k_bar_mathf(int iters, long long* out, uint32_t pp) {  // barrier + 8 dependent FP64 mulmods
  const double p = pp, pinv = 1.0 / pp;
  double a = threadIdx.x + 3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 8; ++j) a = redf(fma(a, a + j, 37.0), p, pinv);
  }
  if (threadIdx.x == 0) out[6] = (clock64() - t0) / iters;
  if (a == 12345.0) out[5] = 1;
}
__global__ void k_thr_int(int iters, long long* out, uint32_t p) {  // throughput: 8 independent red48 chains
  const uint32_t mu32 = 0xffffffffu / p, R = (uint32_t)((1ull << 32) % p);
  uint32_t a[8];
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x + j;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = red48((uint64_t)a[j] * (a[j] + 1) * 37u, mu32, R, p);
  }
  if (threadIdx.x == 0) out[7] = (clock64() - t0) / iters;
  uint32_t s = 0; for (int j = 0; j < 8; ++j) s += a[j]; if (s == 12345) out[5] = s;
}
__global__ void k_thr_f64(int iters, long long* out, uint32_t pp) {  // throughput: 8 independent FP64 chains
  const double p = pp, pinv = 1.0 / pp;
  double a[8];
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x + j;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = redf(fma(a[j], a[j] + 1.0, 37.0), p, pinv);
  }
  if (threadIdx.x == 0) out[4] = (clock64() - t0) / iters;
  double s = 0; for (int j = 0; j < 8; ++j) s += a[j]; if (s == 12345.0) out[5] = 1;
}
int main() {
  long long* d; cudaMalloc(&d, 8 * sizeof(long long)); cudaMemset(d, 0, 64);
  uint16_t* tab; cudaMalloc(&tab, 65536 * 2); cudaMemset(tab, 1, 65536 * 2);
  long long h[8];
  for (int nt : {128, 512, 1024}) {
    for (int rep = 0; rep < 2; ++rep) {
      k_bar<<<1, nt>>>(4096, d); k_bar_smem<<<1, nt>>>(4096, d); k_bar_shfl_tab<<<1, nt>>>(4096, d, tab);
      k_bar_math<<<1, nt>>>(4096, d, 65521);
      k_bar_math32<<<1, nt>>>(4096, d, 65521);
      cudaDeviceSynchronize(); cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
      const long long r32 = h[4];
      k_bar_mathf<<<1, nt>>>(4096, d, 65521);
      k_thr_int<<<1, nt>>>(4096, d, 65521);
      cudaDeviceSynchronize(); cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
      const long long ti = h[7], lf = h[6];
      k_thr_f64<<<1, nt>>>(4096, d, 65521);
      cudaDeviceSynchronize(); cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
      if (rep) printf("threads %4d: chain8: red48 %lld  fp64 %lld | independent8: int %lld  fp64 %lld cycles/iter\n",
                      nt, r32, lf, ti, h[4]);

    }
  }
  return 0;
}
