// Microbenchmark of the 128x128 diagonal-block kernels (one CTA each), checked against a
// host LU mod p.  Build (from the repo root):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo \
//        -I paper_1301_4438_b200/csrc -o tools/micro/diag_bench tools/micro/diag_bench.cu
#define PLUQ_DIAG_TRACE 1
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "pluq_diag.cuh"
#include "pluq_diag2.cuh"
using namespace pluq;

__global__ void invtab_k(uint16_t* tab, ModP mp) {
  const uint32_t a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a < mp.p) tab[a] = a ? (uint16_t)invmod(a, mp) : 0;
}

static void host_lu(std::vector<uint32_t>& a, int n, uint32_t p) {
  ModP mp = ModP::make(p);
  for (int t = 0; t < n; ++t) {
    const uint32_t iv = invmod(a[t * n + t], mp);
    for (int i = t + 1; i < n; ++i) {
      const uint32_t l = (uint32_t)((uint64_t)a[i * n + t] * iv % p);
      a[i * n + t] = l;
      for (int j = t + 1; j < n; ++j)
        a[i * n + j] = (uint32_t)(((uint64_t)a[i * n + j] + (uint64_t)(p - l) * a[t * n + j]) % p);
    }
  }
}

template <typename F>
static float time_it(F launch, uint32_t* d, const uint32_t* d0, size_t bytes, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9f;
  for (int r = 0; r < reps; ++r) {
    cudaMemcpy(d, d0, bytes, cudaMemcpyDeviceToDevice);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  return best * 1e3f;
}

int main(int argc, char** argv) {
  const uint32_t p = argc > 1 ? (uint32_t)atol(argv[1]) : 65521u;
  const int n = 128;
  ModP mp = ModP::make(p);
  std::vector<uint32_t> a(n * n), ref;
  srand(7);
  for (auto& v : a) v = (uint32_t)(((uint64_t)rand() * 2654435761u + rand()) % p);
  ref = a;
  host_lu(ref, n, p);
  uint32_t *d, *d0; int* stop; uint16_t* tab = nullptr;
  cudaMalloc(&d, n * n * 4); cudaMalloc(&d0, n * n * 4); cudaMalloc(&stop, 16);
  cudaMemset(stop, 0, 16);
  cudaMemcpy(d0, a.data(), n * n * 4, cudaMemcpyHostToDevice);
  const bool small = p < 65536;
  if (small) { cudaMalloc(&tab, 65536 * 2); invtab_k<<<(p + 255) / 256, 256>>>(tab, mp); }
  View v{d, n, n, n};
  auto check = [&](const char* name, float us) {
    std::vector<uint32_t> out(n * n);
    cudaMemcpy(out.data(), d, n * n * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < n * n; ++i) bad += out[i] != ref[i];
    cudaError_t e = cudaGetLastError();
    printf("%-28s %8.1f us  mismatches %d  %s\n", name, us, bad, e == cudaSuccess ? "" : cudaGetErrorString(e));
  };
  const size_t dsm = diag_reg_smem(small);
  cudaFuncSetAttribute(diag_reg_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
  cudaFuncSetAttribute(diag_reg_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
  cudaFuncSetAttribute(diag_reg_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
  cudaFuncSetAttribute(diag_reg_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
  if (small) {
    check("diag_reg<small,fwd>", time_it([&] { diag_reg_kernel<true, false><<<1, 512, dsm>>>(v, mp, tab, stop, stop + 1, 0); }, d, d0, n * n * 4, 20));
    check("diag_reg<small,rev>", time_it([&] { diag_reg_kernel<true, true><<<1, 512, dsm>>>(v, mp, tab, stop, stop + 1, 0); }, d, d0, n * n * 4, 20));
  } else {
    check("diag_reg<big,fwd>", time_it([&] { diag_reg_kernel<false, false><<<1, 512, dsm>>>(v, mp, tab, stop, stop + 1, 0); }, d, d0, n * n * 4, 20));
    check("diag_reg<big,rev>", time_it([&] { diag_reg_kernel<false, true><<<1, 512, dsm>>>(v, mp, tab, stop, stop + 1, 0); }, d, d0, n * n * 4, 20));
  }
  const size_t dsm2 = diag_run_smem(small);
  cudaFuncSetAttribute(diag_run_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm2);
  cudaFuncSetAttribute(diag_run_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm2);
  cudaFuncSetAttribute(diag_run_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm2);
  if (small) check("diag_run<small,slowred>", time_it([&] { diag_run_kernel<true, false><<<1, 512, dsm2>>>(v, mp, tab, stop, stop + 1, 0); }, d, d0, n * n * 4, 20));
  cudaFuncSetAttribute(diag_run_kernel<true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm2);
  if (small) check("diag_run<small,full>", time_it([&] { diag_run_kernel<true, true, true><<<1, 512, dsm2>>>(v, mp, tab, stop, stop + 1, 0); }, d, d0, n * n * 4, 20));
  if (small) check("diag_run<small>", time_it([&] { diag_run_kernel<true, true><<<1, 512, dsm2>>>(v, mp, tab, stop, stop + 1, 0); }, d, d0, n * n * 4, 20));
  else check("diag_run<big>", time_it([&] { diag_run_kernel<false, false><<<1, 512, dsm2>>>(v, mp, tab, stop, stop + 1, 0); }, d, d0, n * n * 4, 20));
  if (small) {
    cudaMemcpy(d, d0, n * n * 4, cudaMemcpyDeviceToDevice);
    diag_run_kernel<true, true, true><<<1, 512, dsm2>>>(v, mp, tab, stop, stop + 1, 0);
    long long tr[256];
    cudaMemcpyFromSymbol(tr, g_diag_trace, sizeof(tr));
    printf("publish cadence (cycles since pivot 0; delta):\n");
    for (int t = 0; t < 128; ++t)
      printf("%3d %7lld %5lld | last warp consumed +%lld%s", t, tr[t] - tr[0], t ? tr[t] - tr[t - 1] : 0,
             t < 120 ? tr[128 + t] - tr[t] : 0, (t & 1) ? "\n" : "    ");
  }
  // partial block and a zero pivot
  {
    const int pm = 100, pn = 77;
    std::vector<uint32_t> sub(pm * pn), sref;
    for (int i = 0; i < pm; ++i) for (int j = 0; j < pn; ++j) sub[i * pn + j] = a[i * n + j];
    sref = sub;
    {  // host LU of the rectangular block (min(m, n) pivots)
      ModP q = mp;
      for (int t = 0; t < pn; ++t) {
        const uint32_t iv = invmod(sref[t * pn + t], q);
        for (int i = t + 1; i < pm; ++i) {
          const uint32_t l = (uint32_t)((uint64_t)sref[i * pn + t] * iv % p);
          sref[i * pn + t] = l;
          for (int j = t + 1; j < pn; ++j)
            sref[i * pn + j] = (uint32_t)(((uint64_t)sref[i * pn + j] + (uint64_t)(p - l) * sref[t * pn + j]) % p);
        }
      }
    }
    cudaMemcpy(d, sub.data(), pm * pn * 4, cudaMemcpyHostToDevice);
    View pv{d, pn, pm, pn};
    if (small) diag_run_kernel<true, true><<<1, 512, dsm2>>>(pv, mp, tab, stop, stop + 1, 0);
    else diag_run_kernel<false, false><<<1, 512, dsm2>>>(pv, mp, tab, stop, stop + 1, 0);
    std::vector<uint32_t> out(pm * pn);
    cudaMemcpy(out.data(), d, pm * pn * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < pm * pn; ++i) bad += out[i] != sref[i];
    printf("partial 100x77: mismatches %d %s\n", bad, cudaGetErrorString(cudaGetLastError()));
  }
  {
    // zero pivot at t = 37: make row 37 restricted to columns <= 37 a combination of the rows above
    std::vector<uint32_t> z = a;
    for (int j = 0; j <= 37; ++j) {
      uint64_t sacc = 0;
      for (int i = 0; i < 37; ++i) sacc = (sacc + (uint64_t)(i + 3) * z[i * n + j]) % p;
      z[37 * n + j] = (uint32_t)sacc;
    }
    std::vector<uint32_t> zr = z;
    {  // expected state: factors of the first 37 pivots, trailing block original
      std::vector<uint32_t> w = z;
      ModP q = mp;
      for (int t = 0; t < 37; ++t) {
        const uint32_t iv = invmod(w[t * n + t], q);
        for (int i = t + 1; i < n; ++i) {
          const uint32_t l = (uint32_t)((uint64_t)w[i * n + t] * iv % p);
          w[i * n + t] = l;
          for (int j = t + 1; j < n; ++j)
            w[i * n + j] = (uint32_t)(((uint64_t)w[i * n + j] + (uint64_t)(p - l) * w[t * n + j]) % p);
        }
      }
      for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) if (i < 37 || j < 37) zr[i * n + j] = w[i * n + j];
    }
    cudaMemcpy(d, z.data(), n * n * 4, cudaMemcpyHostToDevice);
    cudaMemset(stop, 0, 16);
    if (small) diag_run_kernel<true, true><<<1, 512, dsm2>>>(v, mp, tab, stop, stop + 1, 5);
    else diag_run_kernel<false, false><<<1, 512, dsm2>>>(v, mp, tab, stop, stop + 1, 5);
    std::vector<uint32_t> out(n * n);
    int hs[4];
    cudaMemcpy(out.data(), d, n * n * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(hs, stop, 16, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < n * n; ++i) bad += out[i] != zr[i];
    printf("zero pivot at 37: mismatches %d stop %d status (%d, %d) %s\n", bad, hs[0], hs[1], hs[2],
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
