// Cycles per step of the rank-1 bulk update forms (one CTA, W warps): 32 x IMAD.WIDE.U32 (64-bit
// lazy accumulators), 64 x IMAD (two 32-bit accumulators per element, w split in 8-bit halves),
// 32 x DFMA.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o imad_bench imad_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_wide(int iters, long long* out, const uint32_t* in) {
  unsigned long long acc[8][4];
  for (int r = 0; r < 8; ++r) for (int q = 0; q < 4; ++q) acc[r][q] = threadIdx.x + r * 4 + q;
  uint32_t c[8], w[4];
  for (int r = 0; r < 8; ++r) c[r] = in[r + threadIdx.x];
  for (int q = 0; q < 4; ++q) w[q] = in[8 + q + threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[r][q] += (unsigned long long)c[r] * w[q];
    c[i & 7] ^= (uint32_t)acc[0][0] & 1;  // keep the loop from being folded
  }
  long long t1 = clock64();
  unsigned long long s = 0;
  for (int r = 0; r < 8; ++r) for (int q = 0; q < 4; ++q) s += acc[r][q];
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  if (s == 12345) out[7] = s;
}
__global__ void k_split(int iters, long long* out, const uint32_t* in) {
  uint32_t a0[8][4], a1[8][4];
  for (int r = 0; r < 8; ++r) for (int q = 0; q < 4; ++q) { a0[r][q] = threadIdx.x + r; a1[r][q] = q; }
  uint32_t c[8], w0[4], w1[4];
  for (int r = 0; r < 8; ++r) c[r] = in[r + threadIdx.x];
  for (int q = 0; q < 4; ++q) { w0[q] = in[8 + q + threadIdx.x] & 255; w1[q] = in[8 + q + threadIdx.x] >> 8; }
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int q = 0; q < 4; ++q) { a0[r][q] += c[r] * w0[q]; a1[r][q] += c[r] * w1[q]; }
    c[i & 7] ^= a0[0][0] & 1;
  }
  long long t1 = clock64();
  uint32_t s = 0;
  for (int r = 0; r < 8; ++r) for (int q = 0; q < 4; ++q) s += a0[r][q] + a1[r][q];
  if (threadIdx.x == 0) out[1] = (t1 - t0) / iters;
  if (s == 12345) out[7] = s;
}
__global__ void k_dfma(int iters, long long* out, const uint32_t* in) {
  double acc[8][4];
  for (int r = 0; r < 8; ++r) for (int q = 0; q < 4; ++q) acc[r][q] = threadIdx.x + r * 4 + q;
  double c[8], w[4];
  for (int r = 0; r < 8; ++r) c[r] = in[r + threadIdx.x];
  for (int q = 0; q < 4; ++q) w[q] = in[8 + q + threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[r][q] = fma(c[r], w[q], acc[r][q]);
    c[i & 7] += acc[0][0] > 1e300 ? 1.0 : 0.0;
  }
  long long t1 = clock64();
  double s = 0;
  for (int r = 0; r < 8; ++r) for (int q = 0; q < 4; ++q) s += acc[r][q];
  if (threadIdx.x == 0) out[2] = (t1 - t0) / iters;
  if (s == 12345.0) out[7] = 1;
}
__global__ void k_dp(int iters, long long* out, const uint32_t* in) {
  int a0[8][4], a1[8][4];
  for (int r = 0; r < 8; ++r) for (int q = 0; q < 4; ++q) { a0[r][q] = threadIdx.x + r; a1[r][q] = q; }
  uint32_t c[8], w[4];
  for (int r = 0; r < 8; ++r) c[r] = in[r + threadIdx.x];
  for (int q = 0; q < 4; ++q) w[q] = in[8 + q + threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int q = 0; q < 4; ++q) { a0[r][q] = __dp2a_lo((int)c[r], (int)w[q], a0[r][q]); a1[r][q] = __dp4a((int)c[r], (int)w[q], a1[r][q]); }
    c[i & 7] ^= a0[0][0] & 1;
  }
  long long t1 = clock64();
  int s = 0;
  for (int r = 0; r < 8; ++r) for (int q = 0; q < 4; ++q) s += a0[r][q] + a1[r][q];
  if (threadIdx.x == 0) out[3] = (t1 - t0) / iters;
  if (s == 12345) out[7] = s;
}
int main() {
  long long* out; uint32_t* in;
  cudaMalloc(&out, 64); cudaMalloc(&in, 4096 * 4);
  cudaMemset(in, 1, 4096 * 4);
  for (int threads : {32, 128, 256, 512}) {
    cudaMemset(out, 0, 64);
    k_wide<<<1, threads>>>(2000, out, in);
    k_split<<<1, threads>>>(2000, out, in);
    k_dfma<<<1, threads>>>(2000, out, in);
    k_dp<<<1, threads>>>(2000, out, in);
    long long h[8];
    cudaMemcpy(h, out, 64, cudaMemcpyDeviceToHost);
    printf("threads %4d: 32 IMAD.WIDE %5lld cyc   64 IMAD %5lld cyc   32 DFMA %5lld cyc   32 dp2a + 32 dp4a %5lld cyc  (%s)\n", threads, h[0], h[1], h[2], h[3],
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
