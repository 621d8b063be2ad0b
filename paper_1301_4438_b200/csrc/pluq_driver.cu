// Host recursion driver + C ABI for the B200 PLUQ-mod-p path.
//
// The driver mirrors Algorithm 1 (/root/reference/pkg/src/pluq/recursive.py:186-256)
// node for node on device-resident data:
//   * nodes that fit in shared memory run whole inside one CTA (pluq_small.cuh);
//   * base-case blocks too large for shared memory run the CTA base case on global
//     memory (pluq_basecase.cuh);
//   * larger nodes are split here: permutations, TRSM and the modular GEMM are
//     launched on the context stream; the host reads back only the ranks and
//     permutations of finished children (one sync per child) because the shapes of
//     F, G, R depend on r1, r2, r3;
//   * an all-zero block short-circuits to (I, I, 0) — bit-exact with the reference,
//     which walks the zero tree and returns identity/0 with no charges.
// OpCounts are charged in the reference's closed forms (kernels.py:1-16) on the host
// for the kernel calls it issues and on the device for work done inside kernels.
#include <cuda.h>
#include <cuda_runtime.h>
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cmath>
#include <cstdio>
#include <functional>
#include <future>
#include <memory>
#include <mutex>
#include <thread>
#include <cstring>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/pluq_b200.h"
#include "pluq_kernels.cuh"
#include <chrono>
#include <cstdio>
#include "pluq_tc_gemm.cuh"

using namespace pluq;

namespace {

struct PluqError : std::runtime_error {
  int code;
  PluqError(int c, const std::string& msg) : std::runtime_error(msg), code(c) {}
};

#define CU(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw PluqError(e_ == cudaErrorMemoryAllocation ? kNoMemory : kCuda,               \
                      std::string(#call) + ": " + cudaGetErrorString(e_));                \
  } while (0)

using Perm = std::vector<int32_t>;

Perm ident(int64_t s) {
  Perm p(s);
  for (int64_t i = 0; i < s; ++i) p[i] = (int32_t)i;
  return p;
}
Perm inverse(const Perm& a) {
  Perm out(a.size());
  for (size_t i = 0; i < a.size(); ++i) out[a[i]] = (int32_t)i;
  return out;
}
bool is_ident(const Perm& a) {
  for (size_t i = 0; i < a.size(); ++i)
    if (a[i] != (int32_t)i) return false;
  return true;
}

// Persistent host worker pool of a context: run(n, fn) calls fn(0..n-1) on the workers and
// the calling thread and returns when all are done.  Used by the host-buffer pipeline to
// convert between the reference's storage dtypes and uint32 residues while DMA runs.
class HostPool {
 public:
  explicit HostPool(int workers) {
    for (int i = 0; i < workers; ++i) th_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return (int)th_.size() + 1; }
  void run(int n, const std::function<void(int)>& fn) {
    if (n <= 0) return;
    {
      std::lock_guard<std::mutex> g(mu_);
      fn_.store(&fn);
      n_.store(n);
      done_ = 0;
      next_.store(0);
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return done_ >= n; });
  }

 private:
  void work() {
    int cnt = 0;
    for (int i; (i = next_.fetch_add(1)) < n_.load();) {
      (*fn_.load())(i);
      ++cnt;
    }
    if (cnt) {
      std::lock_guard<std::mutex> g(mu_);
      done_ += cnt;
      if (done_ >= n_.load()) done_cv_.notify_all();
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      work();
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::atomic<const std::function<void(int)>*> fn_{nullptr};
  std::atomic<int> n_{0}, next_{0};
  int done_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

}  // namespace

struct pluq_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  // pinned staging ring for small host->device uploads (reset after every sync)
  char* pin = nullptr;
  size_t pin_cap = 0, pin_off = 0;
  // result staging of base-case / small-node kernels
  int* d_res = nullptr;
  size_t d_res_cap = 0;
  int* h_res = nullptr;
  size_t h_res_cap = 0;
  unsigned long long* d_counts = nullptr;  // 4 device tallies
  unsigned long long* h_counts = nullptr;
  int* d_flag = nullptr;
  int* d_abort = nullptr;  // residue check of a batch, read back at the end of the call
  // Early download (factor_host, option host_early): rows of the ROOT matrix that the speculative
  // LU has finished are copied back and widened while the factorization is still running.
  std::atomic<int64_t> early_rows{0};          // rows [0, early_rows) of the root are final on the device
  std::atomic<bool> early_invalid{false};      // the final rows were modified again (failure / re-permutation)
  bool early_on = false;                       // factor_host is listening
  bool early_root = false;                     // the node being speculated on is the root matrix
  int64_t early_row0 = 0;                      // global row of the current spec_core view
  std::vector<std::pair<int, int>> early_patches;  // pivot repairs (g, cpos): columns [g, g + cpos] rotated in ALL rows
  int* h_estop = nullptr;                      // pinned stop-flag snapshots, one per publication
  int h_estop_n = 0, h_estop_cap = 0;
  bool attr_cols_set = false, attr_rows_set = false;  // shared-memory attributes of the in-place gathers
  int64_t st_early_chunks = 0;                  // chunks downloaded before the factorization ended (last host call)
  int* h_flag = nullptr;
  int* d_stop = nullptr;     // [stop, k0, t] of the speculative no-pivot path
  int* h_stop = nullptr;
  int64_t spec_block = 128;  // panel width of the speculative blocked LU
  int64_t spec_check = 16;   // host checks the stop flag every this many panels
  int64_t spec_panel = 1024; // outer panel width of the two-level speculative LU
  int64_t spec_panel_big = 2048;        // ... for nodes with at least spec_big_elems entries
  int64_t spec_big_elems = 1ll << 30;   // (cfg5 65536^2: 0.50 -> 0.42 s; cfg3 prefers 1024)
  int64_t spec_repairs = 32;            // speculative LU: most zero pivots repaired by a column rotation
  int* d_zflags = nullptr;   // per-depth "node is nonzero" flags (deferred zero test)
  int* h_zflags = nullptr;
  static constexpr int kMaxDepth = 96;
  // options
  int64_t small_cap = 128 * 128;   // max m*n of a node factored whole by one CTA
  int64_t small_threads = 256;    // CTA size of a host-recursion leaf node
  int64_t batch_threads = 128;    // CTA size of the batched kernels (one matrix per CTA)
  int64_t use_tc = 1;
  int64_t tc_min_dim = 128;        // smallest m, n for the tensor-core GEMM
  int64_t tc_min_k = 32;
  int64_t try_generic = 1;         // speculative no-pivot path for generic-profile blocks
  int64_t time_kernels = 0;        // batched path: time the generic and fallback kernels (adds a sync)
  int64_t inv32 = 1;               // 32-bit inverse table in global memory for primes of 17..25 bits (ModP::itab32)
  int64_t batch_dp = 1;            // 64x64 batch kernel: dp2a version (pluq_kernels.cuh crout_dp_kernel)
  int64_t fixed_kernels = 1;       // shape-specialised generic kernels (64x64) when they apply
  int64_t diag_lazy = 4;           // speculative LU diagonal block: 4 = run-ahead register kernel (pluq_diag2.cuh; full 128-blocks, 512 <= p < 2^16, else 3), 3 = lock-step register kernel (pluq_diag.cuh), 1/2 = lazy smem-image, 0 = Crout
  int64_t lookahead = 1;           // speculative LU: trailing update of panel P overlaps panel P+1
  int64_t la_pair = 1;             // ... and panel P's far update merges into P+1's (one K = 2W GEMM)
  int64_t inner_la = 1;            // speculative LU: look-ahead between the 128-wide blocks of a panel
  int64_t panel_rec = 1;          // speculative LU: recursive (halving) panel factorization instead of 128-block right-looking (1: panels >= 2048 wide, 2: always)
  int64_t gather_inplace = 1;     // column gathers: one in-place pass through shared memory when the span fits
  int64_t la_cap = 0;              // ... this stream's tensor-core GEMMs meanwhile: 0 persistent, 1 la_reserve CTAs, 2 one CTA per tile
  int64_t spec_backup = 2;        // speculative LU: 1 = backup copy of the node, 0 = un-factor in place on failure, 2 = backup below spec_unfactor_elems entries
  int64_t spec_unfactor_elems = 1ll << 28;
  int64_t fin_merge = 1;          // group look-ahead: merged K = W + (g - ps) finishing update after a stop
  int64_t replay_async = 1;       // pivot repair: Alg. 1 replayed on a host thread under the last stop's GPU work
  int64_t host_early = 1;         // host-buffer pipeline: download final rows while the speculative LU still runs
  int64_t la_adapt = 1;           // group look-ahead: SM split between far update and panels chosen per group
  int64_t la_side_solve = 0;      // group look-ahead: U rows of the far columns solved on the side stream
  int64_t la_prio = 0;            // speculative LU: critical path on a greatest-priority stream
  int64_t la_free = 0;            // group look-ahead: far update as one CTA per tile on all SMs (use with la_prio)
  int64_t panel_inv = 1;          // recursive panel: accumulate I - L^-1 of the panel (U12 solves as single GEMMs)
  int64_t la_first_single = 1;    // group look-ahead: the first panel of a node is not grouped
  int64_t la_preinv = 1;          // group look-ahead: I - L11^-1 of a panel formed right after its factorization
  int64_t la_pair_big = 2;        // la_pair for nodes factored with >= 2048-wide panels
  int64_t la_reserve_big = 40;    // la_reserve for those nodes
  int64_t la_reserve = 16;         // SMs left to the critical path while the side GEMM runs
  int64_t host_chunks = 24;        // pipeline depth of the host-buffer batched path
  int64_t chunk_shape = 1;         // host-buffer chunks: 0 = equal, 1 = tent (small first and last)
  int64_t exact_kernel = 1;        // non-generic blocks: 1 = rank-profile kernel, 0 = recursion
  int64_t trace_pipeline = 0;      // print the host-batch pipeline timeline to stderr
  int64_t rpm_lazy = 1;            // rank-profile kernel: lazy-reduction register phases
  int64_t par_trsm = 1;            // speculative LU: the panel's L21 and U12 solves on two streams
  int64_t sym_par = 1;             // rank-profile kernel: parallel symbolic replay (16 warps)
  int64_t tc_trsm = 1;             // 128-wide TRSM as one in-place tensor-core GEMM with I - T^-1
  int64_t pair_leaves = 1;         // exact recursion: F and G leaves concurrently, one readback
  int64_t stream_fb = 4;           // batches: CTAs of the concurrent rank-profile consumer (0: after)
  int64_t stream_fb_spin = 4000000;  // consumer spin bound in cycles (~2 ms) without new work
  int64_t rpm_eager = 1;           // rank-profile kernel, p < 2^16: reduced 32-bit registers (else lazy 64-bit)
  int64_t fb_prefix = 1;           // 64x64 batches: the rank-profile kernel resumes after the generic kernel's pivots
  int64_t tc_trsm_min = 256;       // ... when the solved panel has at least this many rows / columns
  int64_t tc_trsm_big = 4;         // triangles of 256 .. one GEMM pass solved at least this many times as wide: full inverse + one in-place GEMM (0 = off)
  int64_t rpm_threads = 512;       // CTA size of the rank-profile kernel (16 warps: 64 rows in registers)
  int64_t check_inputs = 1;        // device inputs: range-check residues first (field.py:140-147 -> EINVAL)
  bool range_check_pending = false;  // the top node's speculative LU validates in its backup copy
  int64_t pool_keep_mb = 2048;     // the context's memory pool is trimmed to this after every call
  cudaMemPool_t pool = nullptr;    // the context's own stream-ordered pool (not the device default pool)
  int64_t host_threads = 0;        // host-buffer pipeline: conversion threads (0 = hardware threads, <= 32)
  int64_t host_chunk_mb = 64;      // host-buffer pipeline: wire bytes per pinned staging chunk
  int64_t host_wire16 = 1;         // host-buffer pipeline, p <= 2^16: 2-byte wire, widened on the device
  std::unique_ptr<HostPool> hpool;
  // backup of a large node for the speculative LU (restored on failure): kept across calls
  // (one node-sized buffer; 2 bytes per entry when p < 2^16), freed by pluq_release_workspace
  void* node_backup = nullptr;
  size_t node_backup_bytes = 0;
  void* backup_buffer(size_t bytes) {
    if (bytes > node_backup_bytes) {
      sync();
      if (node_backup) CU(cudaFree(node_backup));
      node_backup = nullptr;
      node_backup_bytes = 0;
      CU(cudaMalloc(&node_backup, bytes));
      node_backup_bytes = bytes;
    }
    return node_backup;
  }
  char* ring = nullptr;            // pinned staging ring of the host-buffer pipeline (kRing chunks)
  size_t ring_chunk = 0;
  static constexpr int kRing = 4;
  cudaEvent_t ring_ev[kRing] = {};
  float t_generic_ms = 0.f, t_fallback_ms = 0.f;
  // stats of the last factorization
  int64_t st_launch = 0, st_sync = 0, st_nodes = 0, st_small = 0, st_base = 0, st_tc = 0,
          st_simt = 0, st_zero_skips = 0, st_generic = 0, st_spec_ok = 0, st_spec_fail = 0, st_repairs = 0;
  TcGemm tc;
  // host-batch pipeline resources, created once per context
  cudaStream_t side[6] = {};        // H2D, D2H, 4 exact-kernel streams
  std::vector<cudaEvent_t> evpool;  // timing-disabled events
  int32_t* h_bres = nullptr;        // pinned per-block results (P, Q, rank)
  size_t h_bres_cap = 0;
  uint16_t* d_invtab = nullptr;  // inverse table for invtab_p (p < 2^16)
  unsigned long long* gcount_tab = nullptr;  // generic-profile charges of the last batch shape
  int64_t gcount_key[3] = {-1, -1, -1};
  size_t rpm_smem_set[3] = {0, 0, 0};        // dynamic smem already granted to rpm_pluq_kernel<shape>
  uint32_t invtab_p = 0;

  // ModP with the 32-bit inverse table attached when p has 17..25 bits (option inv32)
  uint32_t* d_invtab32 = nullptr;
  uint32_t invtab32_p = 0;
  size_t invtab32_cap = 0;
  ModP modp(uint32_t p) {
    ModP m = ModP::make(p);
    if (!inv32 || p < 65536u || p > (1u << 25)) return m;
    if (invtab32_p != p) {
      if (invtab32_cap < p) {
        if (d_invtab32) CU(cudaFree(d_invtab32));
        d_invtab32 = nullptr;
        CU(cudaMalloc((void**)&d_invtab32, (size_t)p * sizeof(uint32_t)));
        invtab32_cap = p;
      }
      invtab32_kernel<<<148 * 8, 256, 0, stream>>>(d_invtab32, m);
      check_launch();
      invtab32_p = p;
      CU(cudaStreamSynchronize(stream));  // one-time; the table may be read from other streams
    }
    m.itab32 = d_invtab32;
    return m;
  }

  const uint16_t* invtab(uint32_t p) {
    if (p >= 65536) return nullptr;
    if (invtab_p != p) {
      if (!d_invtab) CU(cudaMalloc((void**)&d_invtab, 65536 * sizeof(uint16_t)));
      invtab_kernel<<<64, 256, 0, stream>>>(d_invtab, ModP::make(p));
      check_launch();
      invtab_p = p;
      CU(cudaStreamSynchronize(stream));  // one-time; the table may be read from other streams
    }
    return d_invtab;
  }

  HostPool& host_pool() {
    if (!hpool) {
      int t = (int)host_threads;
      if (t <= 0) t = (int)std::min<unsigned>(32u, std::max(1u, std::thread::hardware_concurrency()));
      hpool.reset(new HostPool(std::max(0, t - 1)));
    }
    return *hpool;
  }
  char* staging_ring(size_t chunk_bytes) {
    if (chunk_bytes > ring_chunk) {
      if (ring) {
        for (auto e : ring_ev) CU(cudaEventSynchronize(e));
        CU(cudaFreeHost(ring));
      }
      ring = nullptr;
      CU(cudaHostAlloc((void**)&ring, chunk_bytes * kRing, cudaHostAllocDefault));
      ring_chunk = chunk_bytes;
    }
    for (auto& e : ring_ev)
      if (!e) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return ring;
  }

  cudaStream_t* side_streams() {
    if (!side[0]) {
      int lo = 0, hi = 0;
      CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));  // hi = greatest priority (numerically lowest)
      for (int i = 0; i < 6; ++i)  // 2 and 4 carry critical-path solves of the speculative LU
        CU(cudaStreamCreateWithPriority(&side[i], cudaStreamNonBlocking, (i == 2 || i == 4) ? hi : lo));
    }
    return side;
  }
  cudaStream_t hi_stream_ = nullptr;
  cudaStream_t hi_stream() {  // greatest-priority stream for the panel path under a running far update
    if (!hi_stream_) {
      int lo = 0, hi = 0;
      CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      CU(cudaStreamCreateWithPriority(&hi_stream_, cudaStreamNonBlocking, hi));
    }
    return hi_stream_;
  }
  cudaEvent_t* events(size_t count) {
    while (evpool.size() < count) {
      cudaEvent_t e;
      CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      evpool.push_back(e);
    }
    return evpool.data();
  }
  int32_t* batch_results(size_t ints) {
    if (ints > h_bres_cap) {
      if (h_bres) CU(cudaFreeHost(h_bres));
      h_bres_cap = std::max(ints, size_t(1) << 20);
      CU(cudaHostAlloc((void**)&h_bres, h_bres_cap * sizeof(int32_t), cudaHostAllocDefault));
    }
    return h_bres;
  }

  void reset_stats() {
    st_early_chunks = 0;
    st_launch = st_sync = st_nodes = st_small = st_base = st_tc = st_simt = st_zero_skips = st_generic = st_spec_ok =
        st_spec_fail = st_repairs = 0;
    tc.acc_launches = 0;
    tc.acc_ms = tc.acc_ops = 0.0;
  }

  void sync() {
    CU(cudaStreamSynchronize(stream));
    ++st_sync;
    pin_off = 0;
  }
  void* stage(const void* src, size_t bytes) {
    size_t need = (bytes + 255) & ~size_t(255);
    if (pin_off + need > pin_cap) {
      sync();
      if (need > pin_cap) {
        if (pin) CU(cudaFreeHost(pin));
        pin_cap = std::max(need, size_t(16) << 20);
        CU(cudaHostAlloc((void**)&pin, pin_cap, cudaHostAllocDefault));
      }
    }
    void* dst = pin + pin_off;
    pin_off += need;
    std::memcpy(dst, src, bytes);
    return dst;
  }
  void ensure_res(size_t ints) {
    if (ints > d_res_cap) {
      sync();
      if (d_res) CU(cudaFree(d_res));
      if (h_res) CU(cudaFreeHost(h_res));
      d_res_cap = h_res_cap = std::max(ints, size_t(1) << 16);
      CU(cudaMalloc((void**)&d_res, d_res_cap * sizeof(int)));
      CU(cudaHostAlloc((void**)&h_res, h_res_cap * sizeof(int), cudaHostAllocDefault));
    }
  }
  template <class T>
  T* dalloc(size_t count) {
    void* p = nullptr;
    if (count == 0) count = 1;
    CU(cudaMallocFromPoolAsync(&p, count * sizeof(T), pool, stream));
    return reinterpret_cast<T*>(p);
  }
  void dfree(void* p) {
    if (p) CU(cudaFreeAsync(p, stream));
  }
  template <typename T>
  T* dalloc_on(size_t count, cudaStream_t s) {
    void* p = nullptr;
    if (count == 0) count = 1;
    CU(cudaMallocFromPoolAsync(&p, count * sizeof(T), pool, s));
    return reinterpret_cast<T*>(p);
  }
  void dfree_on(void* p, cudaStream_t s) {
    if (p) CU(cudaFreeAsync(p, s));
  }
  void check_launch() {
    ++st_launch;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw PluqError(kCuda, std::string("kernel launch: ") + cudaGetErrorString(e));
  }
};

namespace {

inline int grid_rows(int64_t rows) { return (int)std::max<int64_t>(1, std::min<int64_t>(rows, 65535)); }

struct Ops {
  pluq_ctx* c;
  ModP mp;
  const int* stop = nullptr;  // device stop flag of the speculative path (nullptr: none)
  cudaStream_t st = nullptr;  // stream of this Ops (nullptr: the context's stream)
  int max_ctas = 0;           // cap on the tensor-core GEMM's persistent grid (0: one CTA per SM)
  cudaStream_t s() const { return st ? st : c->stream; }

  // ---- modular GEMM: C <- C - A B  (kernels.py:38-55) ------------------------------
  void gemm(const View& cv, const View& av, const View& bv) {
    if (cv.m == 0 || cv.n == 0 || av.n == 0) return;
    if (c->use_tc && cv.m >= c->tc_min_dim && cv.n >= c->tc_min_dim && av.n >= c->tc_min_k) {
      int st = c->tc.run(cv, av, bv, mp, s(), stop, max_ctas);
      if (st == kOk) { ++c->st_tc; c->st_launch += 3; return; }
      if (st != kUnsupported) throw PluqError(st, "tensor-core GEMM failed: " + c->tc.last_error);
    }
    dim3 grid((cv.n + SG_BN - 1) / SG_BN, (cv.m + SG_BM - 1) / SG_BM);
    if (grid.y > 65535) {  // split very tall C into row chunks
      for (int r0 = 0; r0 < cv.m; r0 += 65535 * SG_BM) {
        int rr = std::min(cv.m - r0, 65535 * SG_BM);
        gemm(cv.sub(r0, 0, rr, cv.n), av.sub(r0, 0, rr, av.n), bv);
      }
      return;
    }
    if (mp.kchunk < 2 * SG_BK)
      simt_gemm_kernel<true><<<grid, 256, 0, s()>>>(cv, av, bv, mp, stop);
    else
      simt_gemm_kernel<false><<<grid, 256, 0, s()>>>(cv, av, bv, mp, stop);
    ++c->st_simt;
    c->check_launch();
  }

  // split point on the 64-grid of the precomputed diagonal-block inverses
  static int split(int r) {
    int nb = (r + TR_BASE - 1) / TR_BASE;
    return TR_BASE * (nb / 2);
  }

  // ---- B <- L^-1 B (kernels.py:59-83) -------------------------------------------------
  // 128 x 128 triangular factor: B' = I - T^-1 from the two 64-block inverses, then one
  // in-place tensor-core GEMM (C aliases an operand; both are split into limb planes first).
  bool trsm128_tc(const View& t, const View& b, bool upper) {
    if (!c->tc_trsm || !c->use_tc || t.m != 128 || (upper ? b.m : b.n) < c->tc_trsm_min) return false;
    uint32_t* inv = c->dalloc_on<uint32_t>(2 * TR_BASE * TR_BASE, s());
    uint32_t* bp = c->dalloc_on<uint32_t>(128 * 128, s());
    if (upper) trinv_upper_kernel<<<2, 256, 0, s()>>>(t, inv, mp, c->invtab(mp.p), stop);
    else trinv_lower_unit_kernel<<<2, 256, 0, s()>>>(t, inv, mp, stop);
    c->check_launch();
    if (upper) trinv128_combine_kernel<true><<<4, 256, 0, s()>>>(t, inv, bp, mp, stop);
    else trinv128_combine_kernel<false><<<4, 256, 0, s()>>>(t, inv, bp, mp, stop);
    c->check_launch();
    const View bpv{bp, 128, 128, 128};
    const int st = upper ? c->tc.run(b, b, bpv, mp, s(), stop, max_ctas) : c->tc.run(b, bpv, b, mp, s(), stop, max_ctas);
    if (st != kOk) throw PluqError(st, "tensor-core TRSM failed: " + c->tc.last_error);
    ++c->st_tc;
    c->st_launch += 3;
    c->dfree_on(bp, s());
    c->dfree_on(inv, s());
    return true;
  }

  // Full inverse X (r x r, pitch r) of the unit-lower (upper = false) or upper triangle t:
  // 64-block inverses on the diagonal, then recursive doubling,
  //   [A 0; B C]^-1 = [A^-1 0; -C^-1 B A^-1  C^-1],  [A B; 0 C]^-1 = [A^-1  -A^-1 B C^-1; 0 C^-1],
  // the off-diagonal blocks as two modular GEMMs each.  ~r^3/3 MACs.
  void tri_inverse(const View& t, bool upper, uint32_t* X) {
    const int r = t.m, nb = (r + TR_BASE - 1) / TR_BASE;
    uint32_t* inv = c->dalloc_on<uint32_t>((size_t)nb * TR_BASE * TR_BASE, s());
    uint32_t* tmp = c->dalloc_on<uint32_t>((size_t)r * ((r + 1) / 2 + TR_BASE), s());
    if (upper) trinv_upper_kernel<<<nb, 256, 0, s()>>>(t, inv, mp, c->invtab(mp.p), stop);
    else trinv_lower_unit_kernel<<<nb, 256, 0, s()>>>(t, inv, mp, stop);
    c->check_launch();
    const View xv{X, r, r, r};
    CU(cudaMemsetAsync(X, 0, (size_t)r * r * sizeof(uint32_t), s()));
    place_blocks_kernel<<<nb, 256, 0, s()>>>(inv, xv, stop);
    c->check_launch();
    for (int b = TR_BASE; b < r; b *= 2)
      for (int j0 = 0; j0 + b < r; j0 += 2 * b) {
        const int b2 = std::min(b, r - j0 - b);
        const View xtt = xv.sub(j0, j0, b, b), xbb = xv.sub(j0 + b, j0 + b, b2, b2);
        if (!upper) {  // X_bt = -X_bb T_bt X_tt
          const View tv{tmp, b, b2, b};
          CU(cudaMemsetAsync(tmp, 0, (size_t)b2 * b * sizeof(uint32_t), s()));
          gemm(tv, t.sub(j0 + b, j0, b2, b), xtt);  // -T_bt X_tt
          negate(tv);
          gemm(xv.sub(j0 + b, j0, b2, b), xbb, tv);
        } else {       // X_tb = -X_tt U_tb X_bb
          const View tv{tmp, b2, b, b2};
          CU(cudaMemsetAsync(tmp, 0, (size_t)b * b2 * sizeof(uint32_t), s()));
          gemm(tv, t.sub(j0, j0 + b, b, b2), xbb);  // -U_tb X_bb
          negate(tv);
          gemm(xv.sub(j0, j0 + b, b, b2), xtt, tv);
        }
      }
    c->dfree_on(tmp, s());
    c->dfree_on(inv, s());
  }
  void negate(const View& v) {
    dim3 grid((v.n + 255) / 256, grid_rows(v.m));
    negate_kernel<<<grid, 256, 0, s()>>>(v, mp, stop);
    c->check_launch();
  }

  // Large triangles (r >= 256, one exact GEMM pass): B <- T^-1 B (or B U^-1) as ONE in-place
  // tensor-core GEMM with I - X, X the full inverse (the operands are split into limb planes
  // before the MMA kernel writes C, so C may alias an operand).  Replaces the recursion whose
  // 64-row SIMT leaves dominated the 2048-wide panel solves of the speculative LU.
  bool trsm_big_tc(const View& t, const View& b, bool upper) {
    const int r = t.m;
    const int L = TcGemm::limbs(mp.p);
    const int wide = upper ? b.m : b.n;
    // the inverse costs ~r^3/3 MACs and ~30 short launches: only worth it for solves much
    // wider than the triangle (cfg5's U rows right of a 2048-wide panel: 61440 x 2048)
    if (!c->tc_trsm_big || !c->use_tc || r < 256 || wide < c->tc_trsm_min || (int64_t)wide < c->tc_trsm_big * r ||
        r > TcGemm::k_pass(L) || c->tc.k_pass_override > 0)
      return false;
    uint32_t* X = c->dalloc_on<uint32_t>((size_t)r * r, s());
    tri_inverse(t, upper, X);
    const View mv{X, r, r, r};
    dim3 grid((r + 255) / 256, grid_rows(r));
    i_minus_kernel<<<grid, 256, 0, s()>>>(mv, upper ? 1 : 0, mp, stop);  // X <- I - X
    c->check_launch();
    const int st = upper ? c->tc.run(b, b, mv, mp, s(), stop, max_ctas) : c->tc.run(b, mv, b, mp, s(), stop, max_ctas);
    if (st != kOk) throw PluqError(st, "tensor-core TRSM failed: " + c->tc.last_error);
    ++c->st_tc;
    c->st_launch += 3;
    c->dfree_on(X, s());
    return true;
  }

  // I - T^-1 of a large triangle computed ahead of its solves (group look-ahead of the
  // speculative LU: the inverse is formed under the running side update, the solves on the
  // critical path are then single GEMMs); nullptr when the one-pass GEMM form does not apply.
  uint32_t* tri_im_inverse(const View& t, bool upper) {
    const int r = t.m;
    const int L = TcGemm::limbs(mp.p);
    if (!c->tc_trsm_big || !c->use_tc || r < 256 || r > TcGemm::k_pass(L) || c->tc.k_pass_override > 0) return nullptr;
    uint32_t* X = c->dalloc_on<uint32_t>((size_t)r * r, s());
    tri_inverse(t, upper, X);
    const View mv{X, r, r, r};
    dim3 grid((r + 255) / 256, grid_rows(r));
    i_minus_kernel<<<grid, 256, 0, s()>>>(mv, upper ? 1 : 0, mp, stop);  // X <- I - X
    c->check_launch();
    return X;
  }
  void trsm_l_pre(uint32_t* X, int r, const View& b) { trsm_l_pre(View{X, r, r, r}, b); }
  void trsm_l_pre(const View& mv, const View& b) {  // B <- L^-1 B = B - (I - L^-1) B, in place
    if (b.n == 0) return;
    const int st = c->tc.run(b, mv, b, mp, s(), stop, max_ctas);
    if (st != kOk) throw PluqError(st, "tensor-core TRSM failed: " + c->tc.last_error);
    ++c->st_tc;
    c->st_launch += 3;
  }

  // I - T^-1 of a 128 x 128 unit-lower block written into a view (pitch ld)
  void tri128_im_lower(const View& t, const View& out) {
    uint32_t* inv = c->dalloc_on<uint32_t>(2 * TR_BASE * TR_BASE, s());
    trinv_lower_unit_kernel<<<2, 256, 0, s()>>>(t, inv, mp, stop);
    c->check_launch();
    trinv128_combine_kernel<false><<<4, 256, 0, s()>>>(t, inv, out.a, mp, stop, (int)out.ld);
    c->check_launch();
    c->dfree_on(inv, s());
  }
  void copy_on(const View& dst, const View& src) {
    if (dst.m == 0 || dst.n == 0) return;
    dim3 grid((dst.n + 255) / 256, grid_rows(dst.m));
    copy_view_kernel<<<grid, 256, 0, s()>>>(dst, src);
    c->check_launch();
  }

  void trsm_l(const View& l, const View& b) {
    const int r = l.m;
    if (r == 0 || b.n == 0) return;
    if (trsm128_tc(l, b, false)) return;
    if (trsm_big_tc(l, b, false)) return;
    const int nb = (r + TR_BASE - 1) / TR_BASE;
    uint32_t* inv = c->dalloc_on<uint32_t>((size_t)nb * TR_BASE * TR_BASE, s());
    trinv_lower_unit_kernel<<<nb, 256, 0, s()>>>(l, inv, mp, stop);
    c->check_launch();
    trsm_l_rec(l, b, inv);
    c->dfree_on(inv, s());
  }
  void trsm_l_rec(const View& l, const View& b, const uint32_t* inv) {
    const int r = l.m;
    if (r <= TR_BASE) {
      trsm_apply_left_kernel<<<(b.n + 31) / 32, 128, 0, s()>>>(inv, b, mp, stop);
      c->check_launch();
      return;
    }
    int h = split(r);
    trsm_l_rec(l.sub(0, 0, h, h), b.sub(0, 0, h, b.n), inv);
    gemm(b.sub(h, 0, r - h, b.n), l.sub(h, 0, r - h, h), b.sub(0, 0, h, b.n));
    trsm_l_rec(l.sub(h, h, r - h, r - h), b.sub(h, 0, r - h, b.n), inv + (size_t)(h / TR_BASE) * TR_BASE * TR_BASE);
  }

  // ---- B <- B U^-1 (kernels.py:85-120) ------------------------------------------------
  void trsm_u(const View& b, const View& u) {
    const int r = u.m;
    if (r == 0 || b.m == 0) return;
    if (trsm128_tc(u, b, true)) return;
    if (trsm_big_tc(u, b, true)) return;
    const int nb = (r + TR_BASE - 1) / TR_BASE;
    uint32_t* inv = c->dalloc_on<uint32_t>((size_t)nb * TR_BASE * TR_BASE, s());
    trinv_upper_kernel<<<nb, 256, 0, s()>>>(u, inv, mp, c->invtab(mp.p), stop);
    c->check_launch();
    trsm_u_rec(b, u, inv);
    c->dfree_on(inv, s());
  }
  void trsm_u_rec(const View& b, const View& u, const uint32_t* inv) {
    const int r = u.m;
    if (r <= TR_BASE) {
      trsm_apply_right_kernel<<<(b.m + 31) / 32, 128, 0, s()>>>(b, inv, mp, stop);
      c->check_launch();
      return;
    }
    int h = split(r);
    trsm_u_rec(b.sub(0, 0, b.m, h), u.sub(0, 0, h, h), inv);
    gemm(b.sub(0, h, b.m, r - h), b.sub(0, 0, b.m, h), u.sub(0, h, h, r - h));
    trsm_u_rec(b.sub(0, h, b.m, r - h), u.sub(h, h, r - h, r - h), inv + (size_t)(h / TR_BASE) * TR_BASE * TR_BASE);
  }

  // ---- un-factoring: partial factors back to the matrix they came from, in place -------
  // C <- C + A B through C <- C - (-A) B (A negated in place and back).
  void gemm_add(const View& cv, const View& av, const View& bv) {
    if (cv.m == 0 || cv.n == 0 || av.n == 0) return;
    negate(av);
    gemm(cv, av, bv);
    negate(av);
  }
  // X <- X U, U upper triangular (g x g), in place: [X1 X2] [Ua Ub; 0 Uc] = [X1 Ua, X1 Ub + X2 Uc].
  void trmm_ru(const View& xv, const View& u) {
    const int g = u.m;
    if (g == 0 || xv.m == 0) return;
    if (g <= TR_BASE) {
      uint32_t* d = c->dalloc_on<uint32_t>(TR_BASE * TR_BASE, s());
      tri_extract_kernel<<<1, 256, 0, s()>>>(u, d, 1);
      c->check_launch();
      trsm_apply_right_kernel<<<(xv.m + 31) / 32, 128, 0, s()>>>(xv, d, mp, stop);  // X <- X D (dense product)
      c->check_launch();
      c->dfree_on(d, s());
      return;
    }
    const int h = split(g);
    trmm_ru(xv.sub(0, h, xv.m, g - h), u.sub(h, h, g - h, g - h));
    gemm_add(xv.sub(0, h, xv.m, g - h), xv.sub(0, 0, xv.m, h), u.sub(0, h, h, g - h));
    trmm_ru(xv.sub(0, 0, xv.m, h), u.sub(0, 0, h, h));
  }
  // Y <- L Y, L unit lower triangular (g x g), in place: [La 0; Lb Lc] [Y1; Y2] = [La Y1; Lb Y1 + Lc Y2].
  void trmm_ll(const View& l, const View& yv) {
    const int g = l.m;
    if (g == 0 || yv.n == 0) return;
    if (g <= TR_BASE) {
      uint32_t* d = c->dalloc_on<uint32_t>(TR_BASE * TR_BASE, s());
      tri_extract_kernel<<<1, 256, 0, s()>>>(l, d, 0);
      c->check_launch();
      trsm_apply_left_kernel<<<(yv.n + 31) / 32, 128, 0, s()>>>(d, yv, mp, stop);  // Y <- D Y
      c->check_launch();
      c->dfree_on(d, s());
      return;
    }
    const int h = split(g);
    trmm_ll(l.sub(h, h, g - h, g - h), yv.sub(h, 0, g - h, yv.n));
    gemm_add(yv.sub(h, 0, g - h, yv.n), l.sub(h, 0, g - h, h), yv.sub(0, 0, h, yv.n));
    trmm_ll(l.sub(0, 0, h, h), yv.sub(0, 0, h, yv.n));
  }
  // X (g x g, packed L\U) <- L U in place.
  void lu_mult(const View& xv) {
    const int g = xv.m;
    if (g == 0) return;
    if (g <= TR_BASE) {
      lu_mult_kernel<<<1, 256, 0, s()>>>(xv, mp);
      c->check_launch();
      return;
    }
    const int h = split(g);
    const View x11 = xv.sub(0, 0, h, h), x12 = xv.sub(0, h, h, g - h), x21 = xv.sub(h, 0, g - h, h),
               x22 = xv.sub(h, h, g - h, g - h);
    lu_mult(x22);               // Lc Uc
    gemm_add(x22, x21, x12);    // + Lb Ub (both still factors)
    trmm_ll(x11, x12);          // La Ub
    trmm_ru(x21, x11);          // Lb Ua
    lu_mult(x11);               // La Ua
  }
  // x = [L11\U11, U12; L21, S] after g pivots of the unpivoted LU (S the Schur complement)
  // back to the matrix it was computed from.
  void unfactor(const View& xv, int g) {
    if (g <= 0) return;
    const int m = xv.m, n = xv.n;
    gemm_add(xv.sub(g, g, m - g, n - g), xv.sub(g, 0, m - g, g), xv.sub(0, g, g, n - g));  // A22 = S + L21 U12
    trmm_ll(xv.sub(0, 0, g, g), xv.sub(0, g, g, n - g));                                  // A12 = L11 U12
    trmm_ru(xv.sub(g, 0, m - g, g), xv.sub(0, 0, g, g));                                  // A21 = L21 U11
    lu_mult(xv.sub(0, 0, g, g));                                                         // A11 = L11 U11
  }

  // ---- gathers restricted to the moved set (matrix.py:249-283) ----------------------
  void gather_rows(const View& x, const Perm& g) {
    if (x.m == 0 || x.n == 0) return;
    std::vector<int32_t> src, dst;
    for (int i = 0; i < x.m; ++i)
      if (g[i] != i) { dst.push_back(i); src.push_back(g[i]); }
    if (dst.empty()) return;
    const int nmv = (int)dst.size();
    int* d_idx = c->dalloc<int>(2 * (size_t)nmv);
    std::vector<int32_t> both(src);
    both.insert(both.end(), dst.begin(), dst.end());
    void* h = c->stage(both.data(), both.size() * 4);
    CU(cudaMemcpyAsync(d_idx, h, both.size() * 4, cudaMemcpyHostToDevice, c->stream));
    if (c->gather_inplace && nmv <= 1536) {  // small moved set: one in-place pass by column strips
      const size_t sm = (size_t)nmv * 32 * sizeof(uint32_t);
      if (sm > 48 * 1024 && !c->attr_rows_set) {
        CU(cudaFuncSetAttribute(rows_inplace_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 1536 * 32 * 4));
        c->attr_rows_set = true;
      }
      const int strips = (x.n + 31) / 32;
      rows_inplace_kernel<<<std::min(strips, c->tc.num_sms() * 8), 256, sm, c->stream>>>(x, d_idx, d_idx + nmv, nmv);
      c->check_launch();
      c->dfree(d_idx);
      return;
    }
    uint32_t* tmp = c->dalloc<uint32_t>((size_t)nmv * x.n);
    dim3 grid((unsigned)std::max(1, std::min(8, (x.n / 4 + 255) / 256)), grid_rows(nmv));
    rows_to_tmp_kernel<<<grid, 256, 0, c->stream>>>(x, d_idx, nmv, tmp);
    c->check_launch();
    tmp_to_rows_kernel<<<grid, 256, 0, c->stream>>>(x, d_idx + nmv, nmv, tmp);
    c->check_launch();
    c->dfree(tmp);
    c->dfree(d_idx);
  }
  void gather_cols(const View& x, const Perm& g) {
    if (x.m == 0 || x.n == 0) return;
    std::vector<int32_t> src, dst;
    for (int j = 0; j < x.n; ++j)
      if (g[j] != j) { dst.push_back(j); src.push_back(g[j]); }
    if (dst.empty()) return;
    const int nmv = (int)dst.size();
    int* d_idx = c->dalloc<int>(2 * (size_t)nmv);
    std::vector<int32_t> both(src);
    both.insert(both.end(), dst.begin(), dst.end());
    void* h = c->stage(both.data(), both.size() * 4);
    CU(cudaMemcpyAsync(d_idx, h, both.size() * 4, cudaMemcpyHostToDevice, c->stream));
    // single in-place pass when a row's moved span fits shared memory and is dense enough
    // that staging the whole span costs no more HBM sectors than the scattered reads
    const int lo = dst.front(), span = dst.back() + 1 - lo;
    const size_t pitch = ((size_t)span + 3) / 4 * 4 + 8;
    if (c->gather_inplace && (int64_t)nmv * 8 >= span && pitch * 4 <= (size_t)220 * 1024) {
      const int nbuf = 2 * pitch * 4 <= (size_t)220 * 1024 ? 2 : 1;
      const size_t sm = nbuf * pitch * 4;
      if (!c->attr_cols_set) {  // per context (= per device), not per process
        CU(cudaFuncSetAttribute(cols_inplace_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        c->attr_cols_set = true;
      }
      const int threads = span >= 8192 ? 1024 : span >= 2048 ? 512 : 256;
      const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(2048 / threads, (size_t)220 * 1024 / (sm + 1024)));
      const int grid1 = std::min(x.m, c->tc.num_sms() * per_sm);
      cols_inplace_kernel<<<grid1, threads, sm, c->stream>>>(x, d_idx, d_idx + nmv, nmv, lo, span, nbuf);
      c->check_launch();
      c->dfree(d_idx);
      return;
    }
    uint32_t* tmp = c->dalloc<uint32_t>((size_t)nmv * x.m);
    dim3 grid((nmv + 255) / 256, grid_rows(x.m));
    cols_to_tmp_kernel<<<grid, 256, 0, c->stream>>>(x, d_idx, nmv, tmp);
    c->check_launch();
    tmp_to_cols_kernel<<<grid, 256, 0, c->stream>>>(x, d_idx + nmv, nmv, tmp);
    c->check_launch();
    c->dfree(tmp);
    c->dfree(d_idx);
  }

  bool nonzero(const View& x) {
    CU(cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
    dim3 grid((unsigned)std::min<int64_t>(4, (x.n + 255) / 256), grid_rows(std::min<int64_t>(x.m, 4096)));
    nonzero_kernel<<<grid, 256, 0, c->stream>>>(x, c->d_flag);
    c->check_launch();
    CU(cudaMemcpyAsync(c->h_flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    return *c->h_flag != 0;
  }

  // Smallest column index of a nonzero entry of the 1 x n view (-1 if the row is zero).
  int first_nonzero_col(const View& x) {
    CU(cudaMemsetAsync(c->d_flag, 0x7f, sizeof(int), c->stream));
    first_nonzero_kernel<<<(unsigned)std::max(1, std::min(148, (x.n + 255) / 256)), 256, 0, c->stream>>>(x, c->d_flag);
    c->check_launch();
    CU(cudaMemcpyAsync(c->h_flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    return *c->h_flag < x.n ? *c->h_flag : -1;
  }

  // Launch the zero test of x into d_zflags[slot] without waiting for it.
  void nonzero_async(const View& x, int slot) {
    CU(cudaMemsetAsync(c->d_zflags + slot, 0, sizeof(int), c->stream));
    dim3 grid((unsigned)std::min<int64_t>(4, (x.n + 255) / 256), grid_rows(std::min<int64_t>(x.m, 4096)));
    nonzero_kernel<<<grid, 256, 0, c->stream>>>(x, c->d_zflags + slot);
    c->check_launch();
  }

  void copy_to16(uint16_t* dst, const View& src, int* bad = nullptr) {
    if (src.m == 0 || src.n == 0) return;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 16, ((int64_t)src.m * src.n / 4 + 255) / 256));
    copy_to16_kernel<<<grid, 256, 0, c->stream>>>(dst, src, mp.p, bad);
    c->check_launch();
  }
  void backup32(uint32_t* dst, const View& src, int* bad) {
    if (src.m == 0 || src.n == 0) return;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 16, ((int64_t)src.m * src.n + 255) / 256));
    backup32_kernel<<<grid, 256, 0, c->stream>>>(dst, src, mp.p, bad);
    c->check_launch();
  }
  void copy_from16(const View& dst, const uint16_t* src) {
    if (dst.m == 0 || dst.n == 0) return;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 16, ((int64_t)dst.m * dst.n / 4 + 255) / 256));
    copy_from16_kernel<<<grid, 256, 0, c->stream>>>(dst, src);
    c->check_launch();
  }
  void copy(const View& dst, const View& src) {
    if (dst.m == 0 || dst.n == 0) return;
    dim3 grid((dst.n + 255) / 256, grid_rows(dst.m));
    copy_view_kernel<<<grid, 256, 0, c->stream>>>(dst, src);
    c->check_launch();
  }
};

// OpCounts of the reference recursion on a matrix with a GENERIC rank profile (leading
// principal minors of orders 1..rho nonzero, Schur complement after rho pivots zero).
// On such inputs every node is again generic with rank min(rows, cols, remaining
// rank), pivots sit on the diagonal and P = Q = I, so the reference's charges
// (kernels.py:1-16, iterative.py:63-75) are a function of (m, n, rho, threshold).
static void generic_counts_rec(int64_t m, int64_t n, int64_t rho, int64_t thr, Counts& c) {
  if (m == 0 || n == 0) return;
  const int64_t rr = std::min(std::min(m, n), rho);
  if (m == 1 || n == 1 || std::min(m, n) <= thr) {
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
  const int64_t r1 = std::min(std::min(kr, kc), rho);
  generic_counts_rec(kr, kc, rho, thr, c);
  charge_trsm_l(c, r1, n - kc);
  charge_trsm_u(c, m - kr, r1);
  charge_mm(c, kr - r1, n - kc, r1);
  charge_mm(c, m - kr, kc - r1, r1);
  charge_mm(c, m - kr, n - kc, r1);
  const int64_t r2 = std::min(std::min(kr - r1, n - kc), rho - r1);
  generic_counts_rec(kr - r1, n - kc, rho - r1, thr, c);
  const int64_t r3 = std::min(std::min(m - kr, kc - r1), rho - r1 - r2);
  generic_counts_rec(m - kr, kc - r1, rho - r1 - r2, thr, c);
  const int64_t m4 = m - kr - r3, n4 = n - kc - r2;
  charge_trsm_u(c, r3, r2);
  charge_trsm_l(c, r3, r2);
  charge_trsm_u(c, m4, r2);
  charge_trsm_l(c, r3, n4);
  charge_mm(c, r3, n4, r2);
  charge_mm(c, m4, n4, r2);
  charge_mm(c, m4, n4, r3);
  generic_counts_rec(m4, n4, rho - r1 - r2 - r3, thr, c);
}


// Per-rank table of generic-profile charges, uploaded for the batched kernel.
// Per-rank closed-form charges of a generic m x n block, on the device.  The table of the
// last (m, n, threshold) is kept in the context (cached: the batch API is called per step).
static unsigned long long* upload_generic_counts(pluq_ctx* c, int64_t m, int64_t n, int64_t thr) {
  if (c->gcount_tab && c->gcount_key[0] == m && c->gcount_key[1] == n && c->gcount_key[2] == thr)
    return c->gcount_tab;
  if (c->gcount_tab) {
    c->sync();
    CU(cudaFree(c->gcount_tab));
    c->gcount_tab = nullptr;
  }
  const int64_t mn = std::min(m, n);
  std::vector<unsigned long long> tab((size_t)(mn + 1) * 4);
  for (int64_t r = 0; r <= mn; ++r) {
    Counts g{0, 0, 0, 0};
    generic_counts_rec(m, n, r, thr, g);
    tab[4 * r] = g.mul; tab[4 * r + 1] = g.add; tab[4 * r + 2] = g.inv; tab[4 * r + 3] = g.red;
  }
  unsigned long long* dt = nullptr;
  CU(cudaMalloc((void**)&dt, tab.size() * sizeof(unsigned long long)));
  CU(cudaMemcpy(dt, tab.data(), tab.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice));
  c->gcount_tab = dt;
  c->gcount_key[0] = m; c->gcount_key[1] = n; c->gcount_key[2] = thr;
  return dt;
}

struct NodeRes {
  Perm P, Q;
  int r;
};

// Block permutations S and T of Algorithm 1 (recursive.py:77-99) as index maps.
static int s_sigma_h(int x, int r1, int r2, int r3, int r4, int k) {
  const int a = r1 + r2, cc = r3 + r4, b = k - a;
  if (x >= a && x < k) return x + cc;
  if (x >= k && x < k + cc) return x - b;
  return x;
}
static int t_sigma_h(int x, int r1, int r2, int r3, int r4, int k) {
  if (x < r1) return x;
  if (x < r1 + r2) return x + (k - r1);
  if (x < r1 + r2 + r3) return x - r2;
  if (x < r1 + r2 + r3 + r4) return x + (k + r2 - (r1 + r2 + r3));
  if (x < k + r2 + r4) return x - (r2 + r4);
  return x;
}

// Algorithm 1 (recursive.py:186-256) with the Algorithm 2 base case (iterative.py:23-91)
// replayed SYMBOLICALLY on a rank profile matrix R_A, on the host, for any size.  The
// device version for single-CTA blocks is sym_rec / sym_base (pluq_rpm.cuh), which states
// the facts this rests on (tests/test_rpm_fallback.py): P, Q, rank and OpCounts of Alg.1 on
// A equal those of Alg.1 on R_A; on a partial permutation every TRSM/GEMM of the recursion
// is the identity on the pattern, so a node only reorders its row/column index lists by
// its children's permutations.  Nodes without a pivot are the identity with no charges.
struct SymHost {
  const std::vector<int>& rp;  // original row -> original column of its one (-1: none)
  const std::vector<int>& cp;  // original column -> original row (-1: none)
  int thr;
  Counts cnt{0, 0, 0, 0};
  std::vector<int> cmark;         // stamp of the current node's column list
  std::vector<int> rpos, cpos;    // local position of an original row / column in a base case
  int stamp = 0;
  // bump stack for the index lists of the recursion (children are processed one after the
  // other, so a node's lists are released when it returns): no allocation per node
  std::vector<int> stack;
  size_t top = 0;
  int* take(size_t k) {
    int* p = stack.data() + top;
    top += k;
    if (top > stack.size()) throw std::runtime_error("symbolic replay: stack overflow");
    return p;
  }

  SymHost(const std::vector<int>& rp_, const std::vector<int>& cp_, int thr_)
      : rp(rp_), cp(cp_), thr(thr_), cmark(cp_.size(), 0), rpos(rp_.size(), -1), cpos(cp_.size(), -1),
        stack(16 * (rp_.size() + cp_.size()) + 1024) {}

  bool has_pivot(const int* rows, const int* cols, int m, int n) {
    ++stamp;
    for (int b = 0; b < n; ++b) cmark[cols[b]] = stamp;
    for (int a = 0; a < m; ++a) {
      const int x = rp[rows[a]];
      if (x >= 0 && cmark[x] == stamp) return true;
    }
    return false;
  }

  // Alg.2 frontier walk (the host twin of sym_base): P[local row] = position, Q[position]
  // = local column, pivots first, then the rest in local order.
  int base(const int* rows, const int* cols, int m, int n, int* P, int* Q) {
    const size_t mark = top;
    for (int a = 0; a < m; ++a) rpos[rows[a]] = a;
    for (int b = 0; b < n; ++b) cpos[cols[b]] = b;
    const int mn = std::min(m, n);
    int* lr = take(m);
    int* lc = take(n);
    int* ro = take(mn);
    int* co = take(mn);
    int* rowpos = take(m);
    int* colpos = take(n);
    for (int a = 0; a < m; ++a) {
      lr[a] = -1;
      const int x = rp[rows[a]];
      if (x >= 0) {
        const int q = cpos[x];
        if (q >= 0 && q < n && cols[q] == x) lr[a] = q;
      }
    }
    for (int b = 0; b < n; ++b) {
      lc[b] = -1;
      const int y = cp[cols[b]];
      if (y >= 0) {
        const int q = rpos[y];
        if (q >= 0 && q < m && rows[q] == y) lc[b] = q;
      }
    }
    int i = 0, j = 0, r = 0;
    while (i < m || j < n) {
      int pr = -1, pc = -1;
      if (j < n && lc[j] >= 0 && lc[j] < i) { pr = lc[j]; pc = j; ++j; }
      else if (i < m && lr[i] >= 0 && lr[i] < j) { pr = i; pc = lr[i]; ++i; }
      else if (i < m && j < n && lr[i] == j) { pr = i; pc = j; ++i; ++j; }
      else { i = std::min(i + 1, m); j = std::min(j + 1, n); continue; }
      ro[r] = pr;
      co[r] = pc;
      ++r;
    }
    for (int k = 0; k < r; ++k) {  // charges of iterative.py:59-75 per pivot
      long long below = m - 1 - ro[k], right = n - 1 - co[k];
      for (int t = 0; t < k; ++t) { below -= ro[t] > ro[k]; right -= co[t] > co[k]; }
      if (below > 0) {
        cnt.inv += 1; cnt.mul += below + below * right; cnt.add += below * right; cnt.red += below + below * right;
      }
    }
    for (int a = 0; a < m; ++a) rowpos[a] = -1;
    for (int b = 0; b < n; ++b) colpos[b] = -1;
    for (int k = 0; k < r; ++k) { rowpos[ro[k]] = k; colpos[co[k]] = k; }
    for (int x = 0, nxt = r; x < m; ++x) P[x] = rowpos[x] >= 0 ? rowpos[x] : nxt++;
    for (int k = 0; k < r; ++k) Q[k] = co[k];
    for (int x = 0, nxt = r; x < n; ++x) if (colpos[x] < 0) Q[nxt++] = x;
    for (int a = 0; a < m; ++a) rpos[rows[a]] = -1;
    for (int b = 0; b < n; ++b) cpos[cols[b]] = -1;
    top = mark;
    return r;
  }

  int rec(const int* rows, const int* cols, int m, int n, int* P, int* Q) {
    if (m == 0 || n == 0 || !has_pivot(rows, cols, m, n)) {
      for (int a = 0; a < m; ++a) P[a] = a;
      for (int b = 0; b < n; ++b) Q[b] = b;
      return 0;
    }
    if (m == 1 || n == 1 || std::min(m, n) <= thr) return base(rows, cols, m, n, P, Q);
    const size_t mark = top;
    const int kr = m / 2, kc = n / 2;
    int* P1 = take(kr);
    int* Q1 = take(kc);
    const int r1 = rec(rows, cols, kr, kc, P1, Q1);
    int* rt = take(kr);
    int* cl = take(kc);
    for (int a = 0; a < kr; ++a) rt[P1[a]] = rows[a];
    for (int t = 0; t < kc; ++t) cl[t] = cols[Q1[t]];
    charge_trsm_l(cnt, r1, n - kc);
    charge_trsm_u(cnt, m - kr, r1);
    charge_mm(cnt, kr - r1, n - kc, r1);
    charge_mm(cnt, m - kr, kc - r1, r1);
    charge_mm(cnt, m - kr, n - kc, r1);
    int* P2 = take(kr - r1);
    int* Q2 = take(n - kc);
    int* P3 = take(m - kr);
    int* Q3 = take(kc - r1);
    const int r2 = rec(rt + r1, cols + kc, kr - r1, n - kc, P2, Q2);
    const int r3 = rec(rows + kr, cl + r1, m - kr, kc - r1, P3, Q3);
    int* hr = take(m - kr);
    int* hc = take(n - kc);
    for (int a = 0; a < m - kr; ++a) hr[P3[a]] = rows[kr + a];
    for (int t = 0; t < n - kc; ++t) hc[t] = cols[kc + Q2[t]];
    const int m4 = m - kr - r3, n4 = n - kc - r2;
    charge_trsm_u(cnt, r3, r2);
    charge_trsm_l(cnt, r3, r2);
    charge_trsm_u(cnt, m4, r2);
    charge_trsm_l(cnt, r3, n4);
    charge_mm(cnt, r3, n4, r2);
    charge_mm(cnt, m4, n4, r2);
    charge_mm(cnt, m4, n4, r3);
    int* P4 = take(m4);
    int* Q4 = take(n4);
    const int r4 = rec(hr + r3, hc + r2, m4, n4, P4, Q4);
    for (int t = 0; t < m; ++t) {
      int y;
      if (t < kr) { const int z = P1[t]; y = z < r1 ? z : r1 + P2[z - r1]; }
      else { const int z = P3[t - kr]; y = kr + (z < r3 ? z : r3 + P4[z - r3]); }
      P[t] = s_sigma_h(y, r1, r2, r3, r4, kr);
    }
    for (int t = 0; t < n; ++t) {
      const int z = t_sigma_h(t, r1, r2, r3, r4, kc);
      int y;
      if (z < kc) { const int w = z < r1 ? z : r1 + Q3[z - r1]; y = Q1[w]; }
      else { const int zz = z - kc; const int w = zz < r2 ? zz : r2 + Q4[zz - r2]; y = kc + Q2[w]; }
      Q[t] = y;
    }
    top = mark;
    return r1 + r2 + r3 + r4;
  }
};

// P (row -> position), Q (position -> column), rank and charges of Alg.1 on the m x n rank
// profile matrix with ones at (prow[k], pcol[k]).
static int symbolic_replay(int m, int n, int thr, const std::vector<int>& prow, const std::vector<int>& pcol,
                           Perm& P, Perm& Q, Counts& cnt) {
  std::vector<int> rp(m, -1), cp(n, -1);
  for (size_t k = 0; k < prow.size(); ++k) { rp[prow[k]] = pcol[k]; cp[pcol[k]] = prow[k]; }
  SymHost sh(rp, cp, thr);
  std::vector<int> rows(m), cols(n);
  for (int a = 0; a < m; ++a) rows[a] = a;
  for (int b = 0; b < n; ++b) cols[b] = b;
  P.assign(m, 0);
  Q.assign(n, 0);
  const int r = sh.rec(rows.data(), cols.data(), m, n, P.data(), Q.data());
  cnt.mul += sh.cnt.mul; cnt.add += sh.cnt.add; cnt.inv += sh.cnt.inv; cnt.red += sh.cnt.red;
  return r;
}

// Exact factorization of the blocks listed in fl/fc (every block of the grid when fl is
// null): the rank-profile kernel (pluq_rpm.cuh) or the field-arithmetic recursion.
// Dynamic shared memory a single-CTA block kernel may request: the 227 KB per-CTA limit
// minus headroom for the kernels' static shared arrays (the symbolic replay's nodes).
constexpr size_t kMaxDynSmem = 227 * 1024 - 4096;
static size_t block_smem_bytes(int64_t m, int64_t n, int64_t thr) {
  return std::max(small_smem_bytes(m, n, thr), rpm_smem_bytes(m, n));
}
static void launch_exact(pluq_ctx* c, const SmallArgs& a, unsigned grid, unsigned threads, const int* fl,
                         const int* fc, cudaStream_t st) {
  if (c->exact_kernel) {
    const unsigned nt = (unsigned)c->rpm_threads;
    const int shape = rpm_shape(a.m, a.n, (int)nt);
    SmallArgs al = a;
    al.lazy = (int)c->rpm_lazy;
    al.eager = (int)c->rpm_eager;
    size_t smem = rpm_smem_bytes(a.m, a.n, (shape == 1 || shape == 2) && al.lazy && nt == 512 && a.invtab != nullptr);
    // parallel symbolic replay: its scratch follows the table when it still fits
    const size_t par_bytes = (size_t)sym_par_words(a.m, a.n) * 4;
    al.sym_par = 0;
    if (c->sym_par && nt >= 512 && smem + par_bytes <= kMaxDynSmem) {
      al.sym_par = 1;
      al.sym_par_off = (int)(smem - rpm_smem_bytes(a.m, a.n, false));
      smem += par_bytes;
    }
    switch (shape) {
      case 1:
        if (smem > c->rpm_smem_set[1]) {
          CU(cudaFuncSetAttribute(rpm_pluq_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
          c->rpm_smem_set[1] = smem;
        }
        rpm_pluq_kernel<1><<<grid, nt, smem, st>>>(al, fl, fc);
        break;
      case 2:
        if (smem > c->rpm_smem_set[2]) {
          CU(cudaFuncSetAttribute(rpm_pluq_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
          c->rpm_smem_set[2] = smem;
        }
        rpm_pluq_kernel<2><<<grid, nt, smem, st>>>(al, fl, fc);
        break;
      default:
        if (smem > c->rpm_smem_set[0]) {
          CU(cudaFuncSetAttribute(rpm_pluq_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
          c->rpm_smem_set[0] = smem;
        }
        rpm_pluq_kernel<0><<<grid, nt, smem, st>>>(al, fl, fc);
    }
  } else {
    const size_t smem = small_smem_bytes(a.m, a.n, a.threshold);
    CU(cudaFuncSetAttribute(small_pluq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    small_pluq_kernel<<<grid, threads, smem, st>>>(a, fl, fc);
  }
  c->check_launch();
}

void check_residues(pluq_ctx* c, const View& x, uint32_t p);

struct Driver {
  pluq_ctx* c;
  ModP mp;
  int threshold;
  Counts host_counts{0, 0, 0, 0};
  Ops ops;

  Driver(pluq_ctx* ctx, uint32_t p, int thr) : c(ctx), mp(ctx->modp(p)), threshold(thr), ops{ctx, ctx->modp(p)} {}

  bool fits_small(int64_t m, int64_t n) const {
    return m * n <= c->small_cap && block_smem_bytes(m, n, threshold) <= kMaxDynSmem;
  }

  int depth = 0;            // depth of the node being processed
  int flagged_depth = -1;   // deepest ancestor slot with a zero test in flight
  bool zero_known[pluq_ctx::kMaxDepth] = {};

  NodeRes readback(int m, int n, int extra = 0) {
    CU(cudaMemcpyAsync(c->h_res, c->d_res, (size_t)(m + n + 1 + extra) * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    if (flagged_depth >= 0)
      CU(cudaMemcpyAsync(c->h_zflags, c->d_zflags, (size_t)(flagged_depth + 1) * sizeof(int),
                         cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    for (int d = 0; d <= flagged_depth; ++d) zero_known[d] = c->h_zflags[d] == 0;
    NodeRes res;
    res.P.assign(c->h_res, c->h_res + m);
    res.Q.assign(c->h_res + m, c->h_res + m + n);
    res.r = c->h_res[m + n];
    return res;
  }

  // Launch the leaf kernels of x on stream st with results at d_res + off (no readback).
  // Layout at off: [P (m) | Q (n) | rank | generic flag | fail count | fail list (1)].
  void launch_leaf(const View& x, size_t off, cudaStream_t st) {
    int* res = c->d_res + off;
    SmallArgs a;
    a.a = x.a; a.lda = x.ld; a.bstride = 0; a.m = x.m; a.n = x.n; a.threshold = threshold; a.mp = mp;
    a.p_out = res; a.q_out = res + x.m; a.r_out = res + x.m + x.n;
    a.cnt_out = c->d_counts; a.cnt_accumulate = 1;
    a.invtab = c->invtab(mp.p);
    a.try_generic = (int)c->try_generic;
    a.try_depth = 1;
    a.generic_counts = nullptr;
    a.generic_flag = a.try_generic ? res + x.m + x.n + 1 : nullptr;
    a.fail_list = nullptr; a.fail_count = nullptr; a.fail_base = 0;
    if (a.try_generic) {
      a.fail_count = res + x.m + x.n + 2;
      a.fail_list = res + x.m + x.n + 3;
      CU(cudaMemsetAsync(a.fail_count, 0, sizeof(int), st));
      const size_t cs = crout_smem_bytes(x.m, x.n);
      CU(cudaFuncSetAttribute(crout_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cs));
      crout_fast_kernel<<<1, (unsigned)c->small_threads, cs, st>>>(a);
      c->check_launch();
    }
    launch_exact(c, a, 1, (unsigned)c->small_threads, a.fail_list, a.fail_count, st);
    ++c->st_small;
  }

  // F and G of Algorithm 1 are independent (disjoint blocks, both only need A1): when
  // both are single-CTA leaves they run concurrently on two streams and come back with
  // ONE readback (recursive.py:211-212).
  void leaf_pair(const View& f, const View& g, NodeRes& F, NodeRes& G) {
    const size_t off2 = ((size_t)f.m + f.n + 4 + 31) & ~size_t(31);
    const size_t tot = off2 + (size_t)g.m + g.n + 4;
    c->ensure_res(tot);
    cudaStream_t side = c->side_streams()[3];
    cudaEvent_t* ev = c->events(2);
    CU(cudaEventRecord(ev[0], c->stream));
    CU(cudaStreamWaitEvent(side, ev[0], 0));
    launch_leaf(f, 0, c->stream);
    launch_leaf(g, off2, side);
    CU(cudaEventRecord(ev[1], side));
    CU(cudaStreamWaitEvent(c->stream, ev[1], 0));
    CU(cudaMemcpyAsync(c->h_res, c->d_res, tot * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    if (flagged_depth >= 0)
      CU(cudaMemcpyAsync(c->h_zflags, c->d_zflags, (size_t)(flagged_depth + 1) * sizeof(int),
                         cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    for (int dd = 0; dd <= flagged_depth; ++dd) zero_known[dd] = c->h_zflags[dd] == 0;
    auto parse = [&](const View& x, size_t off, NodeRes& R) {
      const int* h = c->h_res + off;
      R.P.assign(h, h + x.m);
      R.Q.assign(h + x.m, h + x.m + x.n);
      R.r = h[x.m + x.n];
      if (c->try_generic && h[x.m + x.n + 1]) {  // generic leaf: charges in closed form
        generic_counts_rec(x.m, x.n, R.r, threshold, host_counts);
        ++c->st_generic;
      }
    };
    parse(f, 0, F);
    parse(g, off2, G);
  }

  bool pairable(const View& x) const { return x.m > 0 && x.n > 0 && fits_small(x.m, x.n); }

  NodeRes leaf_small(const View& x) {
    c->ensure_res((size_t)x.m + x.n + 4);
    SmallArgs a;
    a.a = x.a; a.lda = x.ld; a.bstride = 0; a.m = x.m; a.n = x.n; a.threshold = threshold; a.mp = mp;
    a.p_out = c->d_res; a.q_out = c->d_res + x.m; a.r_out = c->d_res + x.m + x.n;
    a.cnt_out = c->d_counts; a.cnt_accumulate = 1;
    a.invtab = c->invtab(mp.p);
    a.try_generic = (int)c->try_generic;
    a.try_depth = 1;
    a.generic_counts = nullptr;           // charged on the host from the readback below
    a.generic_flag = a.try_generic ? c->d_res + x.m + x.n + 1 : nullptr;
    a.fail_list = nullptr; a.fail_count = nullptr; a.fail_base = 0;
    if (a.try_generic) {
      a.fail_count = c->d_res + x.m + x.n + 2;
      a.fail_list = c->d_res + x.m + x.n + 3;
      CU(cudaMemsetAsync(a.fail_count, 0, sizeof(int), c->stream));
    }
    if (a.try_generic) {
      const size_t cs = crout_smem_bytes(x.m, x.n);
      CU(cudaFuncSetAttribute(crout_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cs));
      crout_fast_kernel<<<1, (unsigned)c->small_threads, cs, c->stream>>>(a);
      c->check_launch();
    }
    launch_exact(c, a, 1, (unsigned)c->small_threads, a.fail_list, a.fail_count, c->stream);
    ++c->st_small;
    NodeRes res = readback(x.m, x.n, 1);
    if (a.try_generic && c->h_res[x.m + x.n + 1]) {  // generic leaf: charges in closed form
      generic_counts_rec(x.m, x.n, res.r, threshold, host_counts);
      ++c->st_generic;
    }
    return res;
  }

  NodeRes leaf_global(const View& x) {
    const int m = x.m, n = x.n, mn = std::min(m, n);
    c->ensure_res((size_t)m + n + 1);
    size_t words = (size_t)(m + n + 3) / 4 + 2 * (size_t)mn + m + n + 8;
    int* scratch = c->dalloc<int>(words);
    uint32_t* tmp = c->dalloc<uint32_t>((size_t)m * n);
    BaseArgs a;
    a.x = x; a.mp = mp;
    a.s.prow = reinterpret_cast<uint8_t*>(scratch);
    a.s.pcol = a.s.prow + m;
    int* p = scratch + (m + n + 3) / 4 + 1;
    a.s.rord = p; p += mn;
    a.s.cord = p; p += mn;
    a.s.rowat = p; p += m;
    a.s.colat = p;
    a.tmp = tmp; a.res = c->d_res; a.cnt_out = c->d_counts;
    basecase_global_kernel<<<1, 1024, 0, c->stream>>>(a);
    c->check_launch();
    ++c->st_base;
    c->dfree(tmp);
    c->dfree(scratch);
    return readback(m, n);
  }

  // ---- speculative no-pivot LU of a whole node (generic rank profile) ----------------
  // Blocked right-looking LU with Crout diagonal blocks, fully asynchronous under the
  // device stop flag.  Success conditions are exactly those of crout_generic (pinned
  // against the oracle): no zero pivot, or a first zero pivot at global g after which
  // the whole Schur complement is zero (rank g).  On success P = Q = I and the node
  // holds the unique factors; otherwise the node is restored and the caller recurses.
  // Unpivoted blocked LU of x (see speculative_lu) run until its first zero pivot.  Returns
  // g = min(m, n) if there was none; otherwise g < min(m, n) with x holding exactly the
  // state after g pivots: [L11\U11, U12; L21, S], S = x[g:, g:] the Schur complement, whose
  // (0, 0) entry is 0.
  // Early download: announce that rows [0, rows) of the root are final once the stream gets here,
  // unless the stop flag was raised before (then the solves before this point were skipped).
  struct EarlyPub { pluq_ctx* c; int slot; int64_t rows; };
  static void CUDART_CB early_publish_cb(void* p) {
    EarlyPub* e = static_cast<EarlyPub*>(p);
    if (e->c->h_estop[e->slot] == 0) {
      int64_t cur = e->c->early_rows.load();
      while (cur < e->rows && !e->c->early_rows.compare_exchange_weak(cur, e->rows)) {}
    }
    delete e;
  }
  void early_publish(int64_t local_rows) {
    if (!c->early_on || !c->early_root) return;
    if (c->h_estop_n >= c->h_estop_cap) return;  // out of snapshot slots: just stop announcing
    const int slot = c->h_estop_n++;
    CU(cudaMemcpyAsync(c->h_estop + slot, c->d_stop, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaLaunchHostFunc(c->stream, early_publish_cb, new EarlyPub{c, slot, c->early_row0 + local_rows}));
  }

  // la_prio: the whole critical path runs on a greatest-priority stream (the far updates on
  // default-priority side streams), so its short kernels are dispatched ahead of pending far
  // update CTAs whenever an SM frees up.
  int spec_core(const View& x, int64_t panel_elems) {
    if (!c->la_prio) return spec_core_impl(x, panel_elems);
    cudaStream_t user = c->stream, hi = c->hi_stream();
    cudaEvent_t e0, e1;
    CU(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
    CU(cudaEventRecord(e0, user));
    CU(cudaStreamWaitEvent(hi, e0, 0));
    c->stream = hi;
    int g = 0;
    try {
      g = spec_core_impl(x, panel_elems);
    } catch (...) {
      c->stream = user;
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      throw;
    }
    CU(cudaEventRecord(e1, hi));
    CU(cudaStreamWaitEvent(user, e1, 0));
    c->stream = user;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return g;
  }
  int spec_core_impl(const View& x, int64_t panel_elems) {
    const int m = x.m, n = x.n, mn = std::min(m, n);
    const int BS = (int)c->spec_block;
    // very large nodes amortise a wider outer panel (fewer, longer-K trailing updates)
    const int64_t panel = (c->spec_panel_big > 0 && panel_elems >= c->spec_big_elems) ? c->spec_panel_big
                                                                                       : c->spec_panel;
    const int W = std::max(BS, (int)(panel / BS) * BS);
    // wide-panel nodes (cfg5): group look-ahead with more SMs left to the two hidden panels
    const bool bigw = W >= 2048;
    const int la_pair = (int)(bigw ? c->la_pair_big : c->la_pair);
    const int la_reserve = (int)(bigw ? c->la_reserve_big : c->la_reserve);
    CU(cudaMemsetAsync(c->d_stop, 0, 4 * sizeof(int), c->stream));
    Ops sops = ops;
    sops.stop = c->d_stop;
    const uint16_t* itab = c->invtab(mp.p);
    const bool reg = c->diag_lazy >= 3 && BS <= 128 && (itab != nullptr || mp.kchunk >= 130);
    // run-ahead producer/consumer version (pluq_diag2.cuh): full aligned 128-blocks, 512 <= p < 2^16
    const bool run = reg && c->diag_lazy == 4 && itab != nullptr && mp.p >= 512 && BS == 128 && (x.ld & 3) == 0 &&
                     (reinterpret_cast<uintptr_t>(x.a) & 15) == 0;
    const bool lazy = !reg && c->diag_lazy && BS <= 128;
    const size_t dsm = reg    ? std::max(diag_reg_smem(itab != nullptr), diag_run_smem(itab != nullptr))
                       : lazy ? diag_lazy_smem(itab != nullptr)
                              : diag_fast_smem(BS, itab != nullptr);
    if (reg) {
      CU(cudaFuncSetAttribute(diag_reg_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
      CU(cudaFuncSetAttribute(diag_reg_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
      CU(cudaFuncSetAttribute(diag_run_kernel<true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
    }
    const int lazy_rw = c->diag_lazy == 2 ? 4 : 8;  // rows per warp of diag_lazy_kernel
    if (lazy) {
      CU(cudaFuncSetAttribute(diag_lazy_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
      CU(cudaFuncSetAttribute(diag_lazy_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
    }
    else CU(cudaFuncSetAttribute(diag_crout_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
    bool stopped_early = false;
    int blk = 0;
    // Look-ahead: the outer update of panel P is split into the next panel's columns
    // (critical path, this stream) and the rest, which runs on a side stream with a
    // capped grid while panel P+1 is factored.  The side update is predicated on a
    // snapshot of the stop flag taken at the end of panel P, so a zero pivot found in
    // a later panel leaves it exactly as the sequential schedule would.
    const bool la = c->lookahead != 0;
    cudaStream_t side = c->side_streams()[5];
    const int npanels = (mn + W - 1) / W;
    int* snap = la ? c->dalloc<int>((size_t)npanels + 1) : nullptr;
    cudaEvent_t ev_main = nullptr, ev_side = nullptr;
    if (la) {
      CU(cudaEventCreateWithFlags(&ev_main, cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&ev_side, cudaEventDisableTiming));
    }
    bool side_pending = false, side1_pending = false;
    cudaEvent_t ev_side1 = nullptr;
    CU(cudaEventCreateWithFlags(&ev_side1, cudaEventDisableTiming));
    uint32_t* xg0 = nullptr;  // I - L11^-1 of the open group's first panel
    // Paired far updates: when panel P defers, its far update (rows below panel P+1, columns
    // beyond it) is merged into panel P+1's as ONE K = 2W tensor-core GEMM (per-tile fixed
    // costs of the one-accumulator-set kernel — the TMEM drain and the MMA restart — halve
    // relative to the MMA work); panel P+1's own rows still get P's update eagerly because
    // its U12 needs them.  deferred[P] records it for the finishing step after a stop.
    int defer_ps = -1;
    std::vector<char> deferred((size_t)npanels + 1, 0);
    // la_pair = 2 (group look-ahead, below): first panel of the open group, and which panels
    // opened a group (for the finishing step after a stop in the group's second panel)
    int gfirst = -1;
    std::vector<char> grouped((size_t)npanels + 1, 0);
    // option trace_pipeline: timing events per panel on both streams, printed at the end
    const bool trace = c->trace_pipeline != 0;
    std::vector<std::pair<std::string, cudaEvent_t>> tev;
    std::vector<double> thost;  // host time when each mark was enqueued
    const auto th0 = std::chrono::steady_clock::now();
    auto mark = [&](const std::string& label, cudaStream_t st) {
      if (!trace) return;
      cudaEvent_t e;
      CU(cudaEventCreate(&e));
      CU(cudaEventRecord(e, st));
      tev.emplace_back(label, e);
      thost.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - th0).count());
    };
    cudaStream_t side2 = c->side_streams()[4];
    cudaEvent_t ev_d = nullptr, ev_t = nullptr;
    CU(cudaEventCreateWithFlags(&ev_d, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&ev_t, cudaEventDisableTiming));
    // Inner look-ahead (option inner_la): block j's update of the panel columns beyond block
    // j+1 runs on a third stream while block j+1's diagonal kernel and L21 solve run, predicated
    // on a stop-flag snapshot taken before block j+1 (so a zero pivot there leaves exactly the
    // sequential state); block j+1's U12 solve and update wait for it.
    const bool ila = c->inner_la != 0;
    cudaStream_t side3 = c->side_streams()[2];
    int* isnap = ila ? c->dalloc<int>((size_t)(mn / BS) + npanels + 2) : nullptr;
    cudaEvent_t ev_m3 = nullptr, ev_i3 = nullptr;
    bool in_pending = false;
    if (ila) {
      CU(cudaEventCreateWithFlags(&ev_m3, cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&ev_i3, cudaEventDisableTiming));
    }
    // Panel inverse accumulated by the recursive panel factorization (option panel_inv): M = I - L^-1
    // of the panel's unit-lower triangle, pitch W; leaves write their 128-blocks, nodes the block
    // below them; U12 solves inside the panel and the outer U-row solves are then single GEMMs.
    uint32_t* minv = nullptr;
    int minv_ps = 0;
    bool minv_side = false;
    auto mview = [&](int r0, int c0, int mm, int nn) {
      return View{minv + (size_t)(r0 - minv_ps) * W + (c0 - minv_ps), W, mm, nn};
    };
    auto launch_diag = [&](int k0, int bs) {
      if (run && bs == 128)
        diag_run_kernel<true, true, true><<<1, 512, dsm, c->stream>>>(x.sub(k0, k0, bs, bs), mp, itab, c->d_stop, c->d_stop + 1, k0);
      else if (reg && itab)
        diag_reg_kernel<true><<<1, 512, dsm, c->stream>>>(x.sub(k0, k0, bs, bs), mp, itab, c->d_stop, c->d_stop + 1, k0);
      else if (reg)
        diag_reg_kernel<false><<<1, 512, dsm, c->stream>>>(x.sub(k0, k0, bs, bs), mp, itab, c->d_stop, c->d_stop + 1, k0);
      else if (lazy && lazy_rw == 8)
        diag_lazy_kernel<8><<<1, 512, dsm, c->stream>>>(x.sub(k0, k0, bs, bs), mp, itab, c->d_stop, c->d_stop + 1, k0);
      else if (lazy)
        diag_lazy_kernel<4><<<1, 1024, dsm, c->stream>>>(x.sub(k0, k0, bs, bs), mp, itab, c->d_stop, c->d_stop + 1, k0);
      else
        diag_crout_fast_kernel<<<1, 1024, dsm, c->stream>>>(x.sub(k0, k0, bs, bs), mp, itab, c->d_stop,
                                                c->d_stop + 1, k0);
      c->check_launch();
    };
    // Recursive panel factorization (option panel_rec): the tall panel [c0, c0 + w) is split
    // in halves on the 128-grid — left half, U12 = L11^-1 A12, A22 -= L21 U12 with K = w1,
    // right half — so the panel's updates are a few GEMMs with K up to W/2 instead of one
    // K = 128 update of the rest of the panel per block (4x less traffic over the panel at
    // W = 2048; it matters when the panel runs on the few SMs the side update leaves free).
    // U12 of a node runs on a side stream next to the L21 solve of the left half's last block.
    std::function<bool(int, int)> prec = [&](int c0, int w) -> bool {
      if (w <= BS) {
        launch_diag(c0, w);
        CU(cudaEventRecord(ev_d, c->stream));
        if (minv) {  // I - L^-1 of the block, on the side stream next to the L21 solve
          CU(cudaStreamWaitEvent(side2, ev_d, 0));
          Ops tops = sops;
          tops.st = side2;
          tops.tri128_im_lower(x.sub(c0, c0, w, w), mview(c0, c0, w, w));
          CU(cudaEventRecord(ev_t, side2));
          minv_side = true;
        }
        sops.trsm_u(x.sub(c0 + w, c0, m - c0 - w, w), x.sub(c0, c0, w, w));  // L21, every row below
        const bool check = blk == 0 || (blk + 1) % c->spec_check == 0;
        ++blk;
        if (check) {  // abort early on non-generic input
          CU(cudaMemcpyAsync(c->h_stop, c->d_stop, 3 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
          c->sync();
          if (c->h_stop[0]) { stopped_early = true; return false; }
        }
        return true;
      }
      const int nbk = (w + BS - 1) / BS, w1 = ((nbk + 1) / 2) * BS, w2 = w - w1;
      if (!prec(c0, w1)) return false;
      const View l11 = x.sub(c0, c0, w1, w1), a12 = x.sub(c0, c0 + w1, w1, w2);
      if (minv) {
        // the inverse work of the side stream is ordered there (leaf inverses, node combines);
        // U12 = A12 - (I - L11^-1) A12 as one GEMM with the left half's accumulated inverse
        Ops tops = sops;
        tops.st = side2;
        tops.trsm_l_pre(mview(c0, c0, w1, w1), a12);
        CU(cudaEventRecord(ev_t, side2));
        CU(cudaStreamWaitEvent(c->stream, ev_t, 0));
      } else if (c->par_trsm) {  // after the last diagonal block of the left half (ev_d), not its L21
        CU(cudaStreamWaitEvent(side2, ev_d, 0));
        Ops tops = sops;
        tops.st = side2;
        tops.trsm_l(l11, a12);
        CU(cudaEventRecord(ev_t, side2));
        CU(cudaStreamWaitEvent(c->stream, ev_t, 0));
      } else {
        sops.trsm_l(l11, a12);
      }
      sops.gemm(x.sub(c0 + w1, c0 + w1, m - c0 - w1, w2), x.sub(c0 + w1, c0, m - c0 - w1, w1), a12);
      if (!prec(c0 + w1, w2)) return false;
      if (minv) {
        // M = I - L^-1 of the node from its halves: M21 = Y2 B Y1 = (B - B M1) - M2 (B - B M1),
        // B the block of L below the left half's triangle (final since the left half returned)
        Ops tops = sops;
        tops.st = side2;
        const View bv = x.sub(c0 + w1, c0, w2, w1);
        const View m21 = mview(c0 + w1, c0, w2, w1);
        uint32_t* tmp = c->dalloc_on<uint32_t>((size_t)w2 * w1, side2);
        const View tv{tmp, w1, w2, w1};
        tops.copy_on(tv, bv);
        tops.gemm(tv, bv, mview(c0, c0, w1, w1));              // T = B - B M1
        tops.copy_on(m21, tv);
        tops.gemm(m21, mview(c0 + w1, c0 + w1, w2, w2), tv);   // M21 = T - M2 T
        c->dfree_on(tmp, side2);
        CU(cudaEventRecord(ev_t, side2));
      }
      return true;
    };
    const bool prec_on = c->panel_rec == 2 || (c->panel_rec == 1 && W >= 2048);
    for (int ps = 0; ps < mn && !stopped_early; ps += W) {
      const int pe = std::min(ps + W, mn);
      mark("P" + std::to_string(ps / W) + " inner", c->stream);
      // While a side update runs on (SMs - la_reserve) persistent CTAs, a tensor-core GEMM of
      // this stream launched with a full grid would get only la_reserve SMs for its first
      // CTAs and the rest after the side update ends (persistent CTAs never yield): cap it.
      // la_cap 1: cap it at la_reserve CTAs; 2: one CTA per tile, so it also takes the SMs
      // the side update frees when it ends
      sops.max_ctas = !(side_pending && c->la_cap) ? 0 : c->la_cap == 2 ? -1 : std::max(1, la_reserve);
      uint32_t* panel_m = nullptr;  // I - L11^-1 of this panel when the recursion accumulated it
      if (prec_on) {
        minv = nullptr;
        minv_side = false;
        if (c->panel_inv && c->use_tc && c->tc_trsm && BS == 128 && pe - ps == W && W % 128 == 0 && W >= 256 &&
            W <= TcGemm::k_pass(TcGemm::limbs(mp.p)) && c->tc.k_pass_override <= 0) {
          minv = c->dalloc<uint32_t>((size_t)W * W);
          minv_ps = ps;
          CU(cudaMemsetAsync(minv, 0, (size_t)W * W * sizeof(uint32_t), c->stream));
        }
        prec(ps, pe - ps);
        if (minv && minv_side) CU(cudaStreamWaitEvent(c->stream, ev_t, 0));
        panel_m = minv;
        minv = nullptr;
        if (panel_m && (stopped_early || !(la && la_pair == 2))) {
          c->dfree(panel_m);
          panel_m = nullptr;
        }
      }
      // inner right-looking LU of the panel columns [ps, pe)
      for (int k0 = ps; k0 < pe && !prec_on; k0 += BS, ++blk) {
        const int bs = std::min(BS, pe - k0);
        launch_diag(k0, bs);
        const View b11 = x.sub(k0, k0, bs, bs);
        if (ila && in_pending && !(c->par_trsm && pe - k0 - bs > 0))
          CU(cudaStreamWaitEvent(c->stream, ev_i3, 0));  // U12 below runs on this stream
        if (c->par_trsm && pe - k0 - bs > 0) {
          // L21 and U12 are independent: U12 runs on a side stream next to L21
          CU(cudaEventRecord(ev_d, c->stream));
          CU(cudaStreamWaitEvent(side2, ev_d, 0));
          if (ila && in_pending) CU(cudaStreamWaitEvent(side2, ev_i3, 0));  // rows k0.. right of block j+1
          Ops tops = sops;
          tops.st = side2;
          tops.trsm_l(b11, x.sub(k0, k0 + bs, bs, pe - k0 - bs));                    // U12 (panel)
          CU(cudaEventRecord(ev_t, side2));
          sops.trsm_u(x.sub(k0 + bs, k0, m - k0 - bs, bs), b11);                     // L21
          CU(cudaStreamWaitEvent(c->stream, ev_t, 0));
        } else {
          sops.trsm_u(x.sub(k0 + bs, k0, m - k0 - bs, bs), b11);                     // L21
          sops.trsm_l(b11, x.sub(k0, k0 + bs, bs, pe - k0 - bs));                    // U12 (panel)
        }
        in_pending = false;
        const int nxt = std::min(bs, pe - k0 - bs);  // columns of the next block
        if (ila && pe - k0 - bs > nxt && nxt > 0) {
          sops.gemm(x.sub(k0 + bs, k0 + bs, m - k0 - bs, nxt), x.sub(k0 + bs, k0, m - k0 - bs, bs),
                    x.sub(k0, k0 + bs, bs, nxt));
          CU(cudaMemcpyAsync(isnap + blk, c->d_stop, sizeof(int), cudaMemcpyDeviceToDevice, c->stream));
          CU(cudaEventRecord(ev_m3, c->stream));
          CU(cudaStreamWaitEvent(side3, ev_m3, 0));
          Ops rops = sops;
          rops.st = side3;
          rops.stop = isnap + blk;
          const int cr = k0 + bs + nxt;
          rops.gemm(x.sub(k0 + bs, cr, m - k0 - bs, pe - cr), x.sub(k0 + bs, k0, m - k0 - bs, bs),
                    x.sub(k0, cr, bs, pe - cr));
          CU(cudaEventRecord(ev_i3, side3));
          in_pending = true;
        } else {
          sops.gemm(x.sub(k0 + bs, k0 + bs, m - k0 - bs, pe - k0 - bs), x.sub(k0 + bs, k0, m - k0 - bs, bs),
                    x.sub(k0, k0 + bs, bs, pe - k0 - bs));
        }
        if (blk == 0 || (blk + 1) % c->spec_check == 0) {  // abort early on non-generic input
          CU(cudaMemcpyAsync(c->h_stop, c->d_stop, 3 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
          c->sync();
          if (c->h_stop[0]) { stopped_early = true; break; }
        }
      }
      if (in_pending) {  // the panel's last look-ahead update
        CU(cudaStreamWaitEvent(c->stream, ev_i3, 0));
        in_pending = false;
      }
      if (stopped_early) break;
      // outer step: U rows [ps, pe) right of the panel, then the K = W trailing update
      const View l11 = x.sub(ps, ps, pe - ps, pe - ps);
      if (la && la_pair == 2) {
        // Group look-ahead: panels P, P+1 form a group.  P's outer step touches only P+1's
        // columns (it does NOT wait for the previous group's far update, which keeps running
        // under P's and P+1's factorizations — only for its first part, P+1's columns);
        // P+1's outer step waits for it, finishes the group's U rows for every column right of
        // the group, updates the NEXT panel's columns on this stream (K = 2W) and launches the
        // K = 2W far update on the side: first the columns of the panel after next, then the rest.
        // I - L11^-1 of each panel is formed right after its factorization (under the side
        // update), so the U-row solves on the critical path are single GEMMs.
        const int pidx = ps / W;
        const int ne1 = std::min(pe + W, n);
        uint32_t* xcur = panel_m ? panel_m : (c->la_preinv && pe - ps == W && pe < n) ? sops.tri_im_inverse(l11, false) : nullptr;
        auto solve = [&](uint32_t* X, const View& l, const View& b) {
          if (X && b.n >= c->tc_trsm_min) sops.trsm_l_pre(X, l.m, b);
          else sops.trsm_l(l, b);
        };
        // (the very first panel stays alone, option la_first_single: its K = W far update starts
        // after ONE exposed panel factorization instead of two)
        if (gfirst < 0 && pe < mn && ne1 <= mn && ne1 < n && !(ps == 0 && c->la_first_single)) {  // P: first panel of a group
          mark("P" + std::to_string(pidx) + " outer", c->stream);
          if (side1_pending) {  // P+1's columns came from the first part of the previous far update
            CU(cudaStreamWaitEvent(c->stream, ev_side1, 0));
            side1_pending = false;
          }
          solve(xcur, l11, x.sub(ps, pe, pe - ps, ne1 - pe));
          sops.gemm(x.sub(pe, pe, m - pe, ne1 - pe), x.sub(pe, ps, m - pe, pe - ps), x.sub(ps, pe, pe - ps, ne1 - pe));
          grouped[pidx] = 1;
          gfirst = ps;
          xg0 = xcur;
          continue;
        }
        mark("P" + std::to_string(pidx) + " inner_end", c->stream);  // before the wait for the far update
        if (side_pending) {
          CU(cudaStreamWaitEvent(c->stream, ev_side, 0));
          side_pending = false;
          side1_pending = false;
        }
        sops.max_ctas = 0;
        mark("P" + std::to_string(pidx) + " outer", c->stream);
        const int gs2 = gfirst >= 0 ? gfirst : ps;  // group start (or this panel alone)
        const int gf = gfirst;
        // U rows of the group for the columns [ca, cb): U rows of P, P's contribution to P+1's
        // rows there, then U rows of P+1
        auto outer_cols = [&](Ops& o, int ca, int cb) {
          if (cb <= ca) return;
          auto solve_o = [&](uint32_t* X, const View& l, const View& b) {
            if (X && b.n >= c->tc_trsm_min) o.trsm_l_pre(X, l.m, b);
            else o.trsm_l(l, b);
          };
          if (gf >= 0) {
            const View l0 = x.sub(gf, gf, ps - gf, ps - gf);
            solve_o(xg0, l0, x.sub(gf, ca, ps - gf, cb - ca));
            o.gemm(x.sub(ps, ca, pe - ps, cb - ca), x.sub(ps, gf, pe - ps, ps - gf), x.sub(gf, ca, ps - gf, cb - ca));
          }
          solve_o(xcur, l11, x.sub(ps, ca, pe - ps, cb - ca));
        };
        gfirst = -1;
        const int nn = std::min(pe + W, n);  // the next panel's columns are updated on this stream
        if (pe < mn && nn < n) {
          // critical path: only the next panel's columns; the far columns' U rows are solved on
          // the side stream right before the far update that consumes them (option la_side_solve)
          const bool ss = c->la_side_solve != 0;
          outer_cols(sops, pe, ss ? nn : n);
          if (!ss) early_publish(pe);  // rows < pe: L part and U rows final
          sops.gemm(x.sub(pe, pe, m - pe, nn - pe), x.sub(pe, gs2, m - pe, pe - gs2), x.sub(gs2, pe, pe - gs2, nn - pe));
          CU(cudaMemcpyAsync(snap + pidx, c->d_stop, sizeof(int), cudaMemcpyDeviceToDevice, c->stream));
          CU(cudaEventRecord(ev_main, c->stream));
          CU(cudaStreamWaitEvent(side, ev_main, 0));
          mark("P" + std::to_string(pidx) + " side", side);
          Ops aops = ops;
          aops.st = side;
          aops.stop = snap + pidx;
          // la_free: one CTA per tile (not persistent) on every SM; with la_prio the panel path's
          // kernels are dispatched ahead of the pending tiles as SMs free up
          // Adaptive split of the SMs (option la_adapt, 2048-wide panels): the far update with
          // K = pe - gs2 on (SMs - r) persistent CTAs against the next group's two panel
          // factorizations on the r SMs left.  Fits of the cfg5 traces at r = 24 / 40 / 56
          // (profiles/r2/NOTES.md): T_far(r) = MACs / ((SMs - r) * rate) with rate = 2.55e12
          // field-MAC/s per SM at K = 4096 (2.29e12 at K = 2048) for two-limb primes, and
          // T_panels(r) = 7.9 ms + 483 ms*SM / r for a pair of 2048-wide panels (nearly
          // independent of the row count: the chain is latency-bound); r minimises the larger.
          int resv = la_reserve;
          if (c->la_adapt && bigw && W == 2048) {
            const int sms = c->tc.num_sms();
            const double limbs = (double)TcGemm::limbs(mp.p);
            const double macs = (double)(m - pe) * (double)(n - nn) * (double)(pe - gs2);
            const double rate = (pe - gs2 >= 4096 ? 2.55e12 : 2.29e12) * 4.0 / (limbs * limbs);
            double best = 1e30;
            for (int r = 16; r <= 64; r += 2) {
              const double tf = 1e3 * macs / ((sms - r) * rate), tp = 7.9 + 483.0 / r;
              const double t = std::max(tf, tp);
              if (t < best) { best = t; resv = r; }
            }
          }
          if (trace) fprintf(stderr, "spec %dx%d: P%d far update K=%d on %d SMs (reserve %d)\n", m, n, pidx, pe - gs2, c->tc.num_sms() - resv, resv);
          aops.max_ctas = c->la_free ? -1 : std::max(1, c->tc.num_sms() - resv);
          const int n2 = std::min(nn + W, n);  // first the columns of the panel after next
          if (ss) outer_cols(aops, nn, n2);
          aops.gemm(x.sub(pe, nn, m - pe, n2 - nn), x.sub(pe, gs2, m - pe, pe - gs2), x.sub(gs2, nn, pe - gs2, n2 - nn));
          CU(cudaEventRecord(ev_side1, side));
          side1_pending = true;
          if (n2 < n) {
            if (ss) outer_cols(aops, n2, n);
            aops.gemm(x.sub(pe, n2, m - pe, n - n2), x.sub(pe, gs2, m - pe, pe - gs2), x.sub(gs2, n2, pe - gs2, n - n2));
          }
          // the inverses are last used on the side stream: released there
          if (xg0) c->dfree_on(xg0, side);
          if (xcur) c->dfree_on(xcur, side);
          xg0 = nullptr;
          xcur = nullptr;
          CU(cudaEventRecord(ev_side, side));
          mark("P" + std::to_string(pidx) + " side_end", side);
          side_pending = true;
        } else {
          outer_cols(sops, pe, n);
          early_publish(pe);
          sops.gemm(x.sub(pe, pe, m - pe, n - pe), x.sub(pe, gs2, m - pe, pe - gs2), x.sub(gs2, pe, pe - gs2, n - pe));
        }
        if (xg0) c->dfree(xg0);
        xg0 = nullptr;
        if (xcur) c->dfree(xcur);
        continue;
      }
      if (side_pending) {  // rows [ps, pe) right of this panel came from the previous side update
        CU(cudaStreamWaitEvent(c->stream, ev_side, 0));
        side_pending = false;
      }
      sops.max_ctas = 0;
      const int ne = std::min(pe + W, n);
      const int gs = defer_ps >= 0 ? defer_ps : ps;  // K range [gs, pe): this panel, or the pair
      mark("P" + std::to_string(ps / W) + " outer", c->stream);
      const bool defer_main = la_pair == 3 && defer_ps < 0 && ne < mn && ne + W < n;
      if (la && pe < mn && ne < n && defer_main) {
        // la_pair 3: the deferring panel's remaining work (U rows right of the next panel, the
        // next panel's rows) on this stream, so the next panel factors on an idle GPU
        sops.trsm_l(l11, x.sub(ps, pe, pe - ps, n - pe));
        sops.gemm(x.sub(pe, pe, m - pe, ne - pe), x.sub(pe, ps, m - pe, pe - ps), x.sub(ps, pe, pe - ps, ne - pe));
        sops.gemm(x.sub(pe, ne, ne - pe, n - ne), x.sub(pe, ps, ne - pe, pe - ps), x.sub(ps, ne, pe - ps, n - ne));
        deferred[ps / W] = 1;
        defer_ps = ps;
        continue;
      }
      if (la && pe < mn && ne < n) {
        sops.trsm_l(l11, x.sub(ps, pe, pe - ps, ne - pe));
        sops.gemm(x.sub(pe, pe, m - pe, ne - pe), x.sub(pe, gs, m - pe, pe - gs), x.sub(gs, pe, pe - gs, ne - pe));
        const int pidx = ps / W;
        CU(cudaMemcpyAsync(snap + pidx, c->d_stop, sizeof(int), cudaMemcpyDeviceToDevice, c->stream));
        CU(cudaEventRecord(ev_main, c->stream));
        CU(cudaStreamWaitEvent(side, ev_main, 0));
        mark("P" + std::to_string(ps / W) + " side", side);
        Ops aops = ops;
        aops.st = side;
        aops.stop = snap + pidx;
        aops.max_ctas = std::max(1, c->tc.num_sms() - la_reserve);
        aops.trsm_l(l11, x.sub(ps, ne, pe - ps, n - ne));
        const bool defer = la_pair == 1 && defer_ps < 0 && ne < mn && ne + W < n;
        if (defer) {  // only the next panel's rows now; the rest merges into its update
          aops.gemm(x.sub(pe, ne, ne - pe, n - ne), x.sub(pe, ps, ne - pe, pe - ps), x.sub(ps, ne, pe - ps, n - ne));
          deferred[pidx] = 1;
          defer_ps = ps;
        } else {
          aops.gemm(x.sub(pe, ne, m - pe, n - ne), x.sub(pe, gs, m - pe, pe - gs), x.sub(gs, ne, pe - gs, n - ne));
          defer_ps = -1;
        }
        CU(cudaEventRecord(ev_side, side));
        mark("P" + std::to_string(ps / W) + " side_end", side);
        side_pending = true;
      } else {
        sops.trsm_l(l11, x.sub(ps, pe, pe - ps, n - pe));
        sops.gemm(x.sub(pe, pe, m - pe, n - pe), x.sub(pe, gs, m - pe, pe - gs), x.sub(gs, pe, pe - gs, n - pe));
        defer_ps = -1;
      }
    }
    if (side_pending) CU(cudaStreamWaitEvent(c->stream, ev_side, 0));
    if (xg0) c->dfree(xg0);
    cudaEventDestroy(ev_side1);
    if (in_pending) CU(cudaStreamWaitEvent(c->stream, ev_i3, 0));
    if (ila) {
      c->dfree(isnap);
      cudaEventDestroy(ev_m3);
      cudaEventDestroy(ev_i3);
    }
    if (trace) {
      mark("end", c->stream);
      CU(cudaDeviceSynchronize());
      for (auto& te : tev) {
        float ms = -1.f;
        const cudaError_t er = cudaEventElapsedTime(&ms, tev[0].second, te.second);
        if (er != cudaSuccess) {
          cudaGetLastError();
          ms = -1.f;
        }
        fprintf(stderr, "spec %dx%d W=%d: %-14s %9.3f ms (host %9.3f ms) %s\n", m, n, W, te.first.c_str(), ms,
                thost[&te - &tev[0]] - thost[0], er == cudaSuccess ? "" : cudaGetErrorString(er));
      }
      for (auto& te : tev) cudaEventDestroy(te.second);  // after the loop: tev[0] is the time origin
    }
    cudaEventDestroy(ev_d);
    cudaEventDestroy(ev_t);
    if (la) {
      c->dfree(snap);
      cudaEventDestroy(ev_main);
      cudaEventDestroy(ev_side);
    }
    if (!stopped_early) {
      CU(cudaMemcpyAsync(c->h_stop, c->d_stop, 3 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      c->sync();
    }
    if (!c->h_stop[0]) return mn;
    {
      // first zero pivot at global g = k0 + t inside panel [ps, pe): finish the pivots
      // [k0, g) inside the panel, then [ps, g) for the columns right of it
      const int k0 = c->h_stop[1], t = c->h_stop[2], g = k0 + t;
      const int ps = (k0 / W) * W, pe = std::min(ps + W, mn);
      const int bs = std::min(BS, pe - k0);
      if (ps >= W && deferred[ps / W - 1]) {
        // the previous panel deferred its far update into this panel's: apply it on the rows
        // below this panel (its own rows already have it), columns right of this panel
        ops.gemm(x.sub(pe, pe, m - pe, n - pe), x.sub(pe, ps - W, m - pe, W), x.sub(ps - W, pe, W, n - pe));
      }
      // (fin_merge: when pivots [ps, g) of this panel follow, the rows below g take the first
      // panel's K = W update and this panel's K = g - ps update as ONE GEMM with K = W + g - ps:
      // one pass over the (m - g) x (n - pe) block instead of two)
      const bool fin_merge = c->fin_merge && ps >= W && grouped[ps / W - 1] && pe < n && g > ps;
      if (ps >= W && grouped[ps / W - 1] && pe < n) {
        // group look-ahead, stop in the group's second panel: the first panel's U rows and
        // its contribution to every row below it, right of this panel, are still pending
        const View l0 = x.sub(ps - W, ps - W, W, W);
        ops.trsm_l(l0, x.sub(ps - W, pe, W, n - pe));
        const int rows1 = fin_merge ? g - ps : m - ps;  // merged: only this panel's pivot rows now
        ops.gemm(x.sub(ps, pe, rows1, n - pe), x.sub(ps, ps - W, rows1, W), x.sub(ps - W, pe, W, n - pe));
      }
      if (t > 0 && prec_on) {
        // recursive panel: the block's own columns only; the panel columns right of it follow
        const View b11 = x.sub(k0, k0, t, t);
        ops.trsm_u(x.sub(k0 + bs, k0, m - k0 - bs, t), b11);
        ops.gemm(x.sub(g, g, m - g, k0 + bs - g), x.sub(g, k0, m - g, t), x.sub(k0, g, t, k0 + bs - g));
      } else if (t > 0) {
        const View b11 = x.sub(k0, k0, t, t);
        ops.trsm_u(x.sub(k0 + bs, k0, m - k0 - bs, t), b11);
        ops.trsm_l(b11, x.sub(k0, k0 + bs, t, pe - k0 - bs));
        ops.gemm(x.sub(g, g, m - g, pe - g), x.sub(g, k0, m - g, t), x.sub(k0, g, t, pe - g));
      }
      if (prec_on) {
        // every node of the panel recursion whose LEFT half holds block k0 was skipped under the
        // stop flag: its right half [c0 + w1, c0 + w) has the pivots < c0 only; apply [c0, g)
        int c0 = ps, w = pe - ps;
        while (w > BS) {
          const int nbk = (w + BS - 1) / BS, w1 = ((nbk + 1) / 2) * BS, w2 = w - w1;
          if (k0 < c0 + w1) {
            if (g > c0) {
              const View u12 = x.sub(c0, c0 + w1, g - c0, w2);
              ops.trsm_l(x.sub(c0, c0, g - c0, g - c0), u12);
              ops.gemm(x.sub(g, c0 + w1, m - g, w2), x.sub(g, c0, m - g, g - c0), u12);
            }
            w = w1;
          } else {
            c0 += w1;
            w = w2;
          }
        }
      }
      if (g > ps) {
        ops.trsm_l(x.sub(ps, ps, g - ps, g - ps), x.sub(ps, pe, g - ps, n - pe));
        if (fin_merge)  // L columns [ps - W, g) against U rows [ps - W, g): both contiguous
          ops.gemm(x.sub(g, pe, m - g, n - pe), x.sub(g, ps - W, m - g, W + g - ps), x.sub(ps - W, pe, W + g - ps, n - pe));
        else
          ops.gemm(x.sub(g, pe, m - g, n - pe), x.sub(g, ps, m - g, g - ps), x.sub(ps, pe, g - ps, n - pe));
      }
      return g;
    }
  }

  // Speculative no-pivot LU of a whole node with local pivot REPAIR.  Success conditions
  // (pinned against the oracle): the first zero pivot at g leaves a zero Schur complement
  // (rank g, P = Q = I), or every zero pivot can be repaired by the row-order elimination
  // that defines the rank profile matrix R_A (pluq_rpm.cuh phase a): at a zero pivot (g, g)
  // with S != 0, row g's pivot is its leftmost nonzero column c (all columns < g are
  // eliminated), so column c is rotated to position g (order-preserving, like the
  // reference's rotations, so "leftmost" keeps meaning original order) and the LU resumes
  // on the Schur complement.  The result is the unpivoted LU of A[:, sigma] with
  // R_A = {(k, sigma[k])}; Alg.1 replayed symbolically on R_A (SymHost) must then give
  // P = I and Q = sigma — by fact (2) the packed output is exactly the reference's — and
  // its charges.  A row with no pivot (row g of S zero), too many repairs, or a replay that
  // disagrees restores the node from the backup and the caller recurses exactly.
  // Returns 0 = failed (x restored), 1 = generic (P = Q = I), 2 = repaired (p_out — empty
  // for the identity — q and cnt set).
  int speculative_lu(const View& x, int& rank, Perm& p_out, Perm& q, Counts& cnt) {
    const int m = x.m, n = x.n, mn = std::min(m, n);
    const bool b16 = mp.p <= 65536u;  // residues fit 16 bits: half the backup traffic
    // spec_backup = 0: no backup copy of the node; a failed speculation is undone by
    // re-multiplying the partial factors in place (Ops::unfactor) and undoing the repairs'
    // column rotations.  Extra storage then stays O(panel) instead of O(m n).
    const bool use_backup = c->spec_backup == 1 || (c->spec_backup == 2 && (int64_t)m * n < c->spec_unfactor_elems);
    void* backup = use_backup ? c->backup_buffer((size_t)m * n * (b16 ? 2 : 4)) : nullptr;
    View bk{static_cast<uint32_t*>(backup), n, m, n};
    // the backup copy doubles as the deferred input range check of the top node (pluq_factor)
    const bool check = c->range_check_pending;
    c->range_check_pending = false;
    if (check && use_backup) CU(cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
    auto save = [&]() {
      if (b16) ops.copy_to16(static_cast<uint16_t*>(backup), x, check ? c->d_flag : nullptr);
      else if (check) ops.backup32(static_cast<uint32_t*>(backup), x, c->d_flag);
      else ops.copy(bk, x);
    };
    Perm sig = ident(n);
    int g_state = 0;  // pivots of the partial factorization currently held in x
    auto restore = [&]() {
      if (use_backup) {
        b16 ? ops.copy_from16(x, static_cast<const uint16_t*>(backup)) : ops.copy(x, bk);
        return;
      }
      ops.unfactor(x, g_state);
      if (!is_ident(sig)) ops.gather_cols(x, inverse(sig));  // column k holds original column sig[k]
      g_state = 0;
    };
    if (use_backup) {
      save();
      if (check) {  // nothing was modified yet
        CU(cudaMemcpyAsync(c->h_flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        if (*c->h_flag) throw PluqError(kInvalid, "matrix entries must be canonical residues in [0, p)");
      }
    } else if (check) {
      check_residues(c, x, mp.p);
    }
    int g0 = 0, repairs = 0, res = 0;
    c->early_root = c->early_on && depth == 0;
    // option trace_pipeline: host-clock phase times of this function (device synchronised at each mark)
    const bool ptrace = c->trace_pipeline != 0;
    auto tp0 = std::chrono::steady_clock::now();
    auto phase = [&](const char* what) {
      if (!ptrace) return;
      CU(cudaDeviceSynchronize());
      const auto t1 = std::chrono::steady_clock::now();
      fprintf(stderr, "spec_lu %dx%d: %-22s %8.3f ms\n", m, n, what, std::chrono::duration<double, std::milli>(t1 - tp0).count());
      tp0 = t1;
    };
    phase("backup / range check");
    struct ReplayOut { Perm P, Q; Counts sc{0, 0, 0, 0}; int rank = -1; };
    ReplayOut pre;  // replay finished under the last stop's GPU work
    for (;;) {
      c->early_row0 = g0;
      const int g = g0 + spec_core(x.sub(g0, g0, m - g0, n - g0), (int64_t)m * n);
      phase("spec_core + finishing");
      // The host is about to wait ~15-20 ms for the finishing GEMMs and the zero test of S: if this
      // stop ends the factorization (S = 0 or g = min(m, n)) the rank is g, so Alg. 1 is replayed on
      // R_A = {(k, sig[k]), k < g} on a host thread meanwhile (6 ms at cfg5); discarded otherwise.
      std::future<ReplayOut> fut;
      if (repairs > 0 && c->replay_async) {
        const int rg = std::min(g, mn), thr = threshold;
        Perm sig_copy = sig;
        fut = std::async(std::launch::async, [rg, m, n, thr, sig_copy]() {
          ReplayOut r;
          std::vector<int> prow(rg), pcol(rg);
          for (int k = 0; k < rg; ++k) { prow[k] = k; pcol[k] = sig_copy[k]; }
          symbolic_replay(m, n, thr, prow, pcol, r.P, r.Q, r.sc);
          r.rank = rg;
          return r;
        });
      }
      g_state = std::min(g, mn);
      if (g >= mn) { rank = mn; res = 1; if (fut.valid()) pre = fut.get(); break; }
      const bool nzs = ops.nonzero(x.sub(g, g, m - g, n - g));
      phase("zero test of S");
      if (!nzs) { rank = g; res = 1; if (fut.valid()) pre = fut.get(); break; }
      if (repairs >= c->spec_repairs) break;
      const int cpos = ops.first_nonzero_col(x.sub(g, g, 1, n - g));
      if (cpos <= 0) break;  // row g has no pivot (rows would move): exact recursion
      ++repairs;
      if (c->early_root) c->early_patches.emplace_back(g, cpos);
      Perm rot(cpos + 1);
      rot[0] = cpos;
      for (int j = 1; j <= cpos; ++j) rot[j] = j - 1;
      ops.gather_cols(x.sub(0, g, m, cpos + 1), rot);
      std::rotate(sig.begin() + g, sig.begin() + g + cpos, sig.begin() + g + cpos + 1);
      phase("repair (rotate column)");
      g0 = g;
    }
    if (res == 1 && repairs > 0) {
      std::vector<int> prow(rank), pcol(rank);
      for (int k = 0; k < rank; ++k) { prow[k] = k; pcol[k] = sig[k]; }
      Perm P, Q;
      Counts sc{0, 0, 0, 0};
      if (pre.rank == rank) {
        P.swap(pre.P);
        Q.swap(pre.Q);
        sc = pre.sc;
      } else {
        symbolic_replay(m, n, threshold, prow, pcol, P, Q, sc);
      }
      phase("symbolic replay (host)");
      res = 2;
      cnt = sc;
      if (is_ident(P) && Q == sig) {
        q = sig;
      } else {
        // Alg.1 orders these pivots differently from row order (e.g. a repair wider than
        // one column inside a base case): R_A is still exact, so the packed output is the
        // unpivoted LU of A' = A[P^-1][:, Q], whose leading minors 1..r are nonzero (fact 2):
        // restore, permute, and factor A' without pivoting.
        if (c->early_root) c->early_invalid.store(true);
        restore();
        ops.gather_rows(x, inverse(P));
        ops.gather_cols(x, Q);
        const int g2 = spec_core(x, (int64_t)m * n);
        if (g2 != rank || (g2 < mn && ops.nonzero(x.sub(g2, g2, m - g2, n - g2))))
          throw PluqError(kCuda, "internal: LU of the rank-profile permuted node is not generic");
        p_out = P;
        q = Q;
      }
    }
    if (res) {
      ++c->st_spec_ok;
      c->st_repairs += repairs;
    } else {
      if (c->early_root) c->early_invalid.store(true);
      restore();
      ++c->st_spec_fail;
    }
    c->early_root = false;
    return res;
  }

  bool spec_disabled = false;

  NodeRes rec(const View& x) {
    const int m = x.m, n = x.n;
    ++c->st_nodes;
    if (m == 0 || n == 0) return NodeRes{ident(m), ident(n), 0};
    const bool base = m == 1 || n == 1 || std::min(m, n) <= threshold;
    if (fits_small(m, n)) return leaf_small(x);
    if (base) return leaf_global(x);
    if (c->try_generic && !spec_disabled) {
      int rk = 0;
      Perm pp, q;
      Counts sc{0, 0, 0, 0};
      const int how = speculative_lu(x, rk, pp, q, sc);
      if (how == 1) {
        generic_counts_rec(m, n, rk, threshold, host_counts);
        return NodeRes{ident(m), ident(n), rk};
      }
      if (how == 2) {
        host_counts.mul += sc.mul; host_counts.add += sc.add; host_counts.inv += sc.inv; host_counts.red += sc.red;
        return NodeRes{pp.empty() ? ident(m) : pp, q, rk};
      }
      spec_disabled = true;  // non-generic node: do not speculate again inside its subtree
      NodeRes res = rec_exact(x);
      spec_disabled = false;
      return res;
    }
    return rec_exact(x);
  }

  NodeRes rec_exact(const View& x) {
    const int m = x.m, n = x.n;
    // Zero-block short-circuit without a dedicated sync: the test result travels back
    // with the next leaf readback (inside A1's subtree).  Factoring A1 of a zero block
    // is exact (identity, r=0, data untouched), so only the left spine is spent.
    const int slot = depth;
    const bool flag_here = slot < pluq_ctx::kMaxDepth;
    if (flag_here) {
      ops.nonzero_async(x, slot);
      flagged_depth = std::max(flagged_depth, slot);
      zero_known[slot] = false;
    } else if (!ops.nonzero(x)) {
      ++c->st_zero_skips;
      return NodeRes{ident(m), ident(n), 0};
    }
    const int kr = m / 2, kc = n / 2;
    ++depth;
    NodeRes A1 = rec(x.sub(0, 0, kr, kc));
    --depth;
    if (flag_here) {
      flagged_depth = std::min(flagged_depth, slot - 1);
      if (zero_known[slot]) {
        ++c->st_zero_skips;
        return NodeRes{ident(m), ident(n), 0};
      }
    }
    const int r1 = A1.r;
    ops.gather_rows(x.sub(0, kc, kr, n - kc), inverse(A1.P));
    ops.gather_cols(x.sub(kr, 0, m - kr, kc), A1.Q);
    ops.trsm_l(x.sub(0, 0, r1, r1), x.sub(0, kc, r1, n - kc));            // D
    ops.trsm_u(x.sub(kr, 0, m - kr, r1), x.sub(0, 0, r1, r1));            // E
    ops.gemm(x.sub(r1, kc, kr - r1, n - kc), x.sub(r1, 0, kr - r1, r1), x.sub(0, kc, r1, n - kc));  // F
    ops.gemm(x.sub(kr, r1, m - kr, n - r1), x.sub(kr, 0, m - kr, r1), x.sub(0, r1, r1, n - r1));    // G|H
    charge_trsm_l(host_counts, r1, n - kc);
    charge_trsm_u(host_counts, m - kr, r1);
    charge_mm(host_counts, kr - r1, n - kc, r1);
    charge_mm(host_counts, m - kr, kc - r1, r1);
    charge_mm(host_counts, m - kr, n - kc, r1);

    ++depth;
    NodeRes F, G;
    {
      const View fv = x.sub(r1, kc, kr - r1, n - kc), gv = x.sub(kr, r1, m - kr, kc - r1);
      if (c->pair_leaves && pairable(fv) && pairable(gv)) {
        c->st_nodes += 2;
        leaf_pair(fv, gv, F, G);
      } else {
        F = rec(fv);
        G = rec(gv);
      }
    }
    const int r2 = F.r;
    const int r3 = G.r;
    --depth;
    {
      Perm ip3 = inverse(G.P), ip2 = inverse(F.P);
      ops.gather_rows(x.sub(kr, kc, m - kr, n - kc), ip3);
      ops.gather_cols(x.sub(kr, kc, m - kr, n - kc), F.Q);
      ops.gather_rows(x.sub(kr, 0, m - kr, r1), ip3);
      ops.gather_rows(x.sub(r1, 0, kr - r1, r1), ip2);
      ops.gather_cols(x.sub(0, kc, r1, n - kc), F.Q);
      ops.gather_cols(x.sub(0, r1, r1, kc - r1), G.Q);
    }
    const View u2 = x.sub(r1, kc, r2, r2);
    const View l3 = x.sub(kr, r1, r3, r3);
    const int m4 = m - kr - r3, n4 = n - kc - r2;
    ops.trsm_u(x.sub(kr, kc, r3, r2), u2);                                  // I
    if (r3 > 0 && r2 > 0) {
      uint32_t* jbuf = c->dalloc<uint32_t>((size_t)r3 * r2);
      View J{jbuf, r2, r3, r2};
      ops.copy(J, x.sub(kr, kc, r3, r2));
      ops.trsm_l(l3, J);                                                    // J (scratch)
      ops.trsm_u(x.sub(kr + r3, kc, m4, r2), u2);                           // K
      ops.trsm_l(l3, x.sub(kr, kc + r2, r3, n4));                           // N
      ops.gemm(x.sub(kr, kc + r2, r3, n4), J, x.sub(r1, kc + r2, r2, n4));  // O
      c->dfree(jbuf);
    } else {
      ops.trsm_u(x.sub(kr + r3, kc, m4, r2), u2);
      ops.trsm_l(l3, x.sub(kr, kc + r2, r3, n4));
    }
    ops.gemm(x.sub(kr + r3, kc + r2, m4, n4), x.sub(kr + r3, kc, m4, r2), x.sub(r1, kc + r2, r2, n4));
    ops.gemm(x.sub(kr + r3, kc + r2, m4, n4), x.sub(kr + r3, r1, m4, r3), x.sub(kr, kc + r2, r3, n4));
    charge_trsm_u(host_counts, r3, r2);
    charge_trsm_l(host_counts, r3, r2);
    charge_trsm_u(host_counts, m4, r2);
    charge_trsm_l(host_counts, r3, n4);
    charge_mm(host_counts, r3, n4, r2);
    charge_mm(host_counts, m4, n4, r2);
    charge_mm(host_counts, m4, n4, r3);

    ++depth;
    NodeRes R = rec(x.sub(kr + r3, kc + r2, m4, n4));
    --depth;
    const int r4 = R.r;
    ops.gather_rows(x.sub(kr + r3, 0, m4, kc + r2), inverse(R.P));
    ops.gather_cols(x.sub(0, kc + r2, kr + r3, n4), R.Q);

    Perm S(m), T(n);
    for (int t = 0; t < m; ++t) S[t] = s_sigma_h(t, r1, r2, r3, r4, kr);
    for (int t = 0; t < n; ++t) T[t] = t_sigma_h(t, r1, r2, r3, r4, kc);
    if (!is_ident(S)) ops.gather_rows(x, inverse(S));
    if (!is_ident(T)) ops.gather_cols(x, T);

    NodeRes out;
    out.P.resize(m);
    out.Q.resize(n);
    for (int t = 0; t < m; ++t) {
      int y;
      if (t < kr) { int z = A1.P[t]; y = z < r1 ? z : r1 + F.P[z - r1]; }
      else { int z = G.P[t - kr]; y = kr + (z < r3 ? z : r3 + R.P[z - r3]); }
      out.P[t] = S[y];
    }
    for (int t = 0; t < n; ++t) {
      int z = T[t], y;
      if (z < kc) { int w = z < r1 ? z : r1 + G.Q[z - r1]; y = A1.Q[w]; }
      else { int zz = z - kc; int w = zz < r2 ? zz : r2 + R.Q[zz - r2]; y = kc + F.Q[w]; }
      out.Q[t] = y;
    }
    out.r = r1 + r2 + r3 + r4;
    return out;
  }

};

int validate(int64_t m, int64_t n, int64_t p) {
  if (m < 0 || n < 0 || m > INT32_MAX / 2 || n > INT32_MAX / 2) return kInvalid;
  if (p < 2 || p >= (int64_t(1) << 31)) return kInvalid;
  return kOk;
}

// Restores the caller's current device on scope exit (the ABI must not change it).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) {
      cudaError_t e = cudaSetDevice(dev);
      if (e != cudaSuccess) throw PluqError(kCuda, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    }
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

template <class F>
int guarded(pluq_ctx* ctx, F&& f) {
  if (!ctx) return kInvalid;
  try {
    DeviceGuard dg(ctx->device);
    f();
    if (ctx->pool) cudaMemPoolTrimTo(ctx->pool, (size_t)std::max<int64_t>(0, ctx->pool_keep_mb) << 20);
    return kOk;
  } catch (const PluqError& e) {
    ctx->err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    ctx->err = "host out of memory";
    return kNoMemory;
  } catch (const std::exception& e) {
    ctx->err = e.what();
    return kCuda;
  }
}

// PLUQ_EINVAL unless every entry of the device view is a canonical residue in [0, p): the
// reference rejects such input when the DenseMatrix is built (field.py:140-147, ValueError),
// before anything is modified.  One read of the view (HBM-bound).
void check_residues(pluq_ctx* c, const View& x, uint32_t p) {
  if (!c->check_inputs || x.m <= 0 || x.n <= 0) return;
  CU(cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
  const int n4 = std::max(1, x.n / 4);
  dim3 grid((unsigned)std::min(4, (n4 + 255) / 256), (unsigned)std::min(x.m, 4096));
  range_check_kernel<<<grid, 256, 0, c->stream>>>(x, p, c->d_flag);
  c->check_launch();
  CU(cudaMemcpyAsync(c->h_flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  if (*c->h_flag) throw PluqError(kInvalid, "matrix entries must be canonical residues in [0, p)");
}

void finish_counts(pluq_ctx* c, const Counts& hc, int64_t* counts) {
  CU(cudaMemcpyAsync(c->h_counts, c->d_counts, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  if (counts) {
    counts[0] += (int64_t)(hc.mul + c->h_counts[0]);
    counts[1] += (int64_t)(hc.add + c->h_counts[1]);
    counts[2] += (int64_t)(hc.inv + c->h_counts[2]);
    counts[3] += (int64_t)(hc.red + c->h_counts[3]);
  }
}

void factor_device(pluq_ctx* c, uint32_t* dA, int64_t ld, int64_t m, int64_t n, int64_t p,
                   int64_t threshold, int64_t* psig, int64_t* qsig, int64_t* rank, int64_t* counts,
                   bool iterative) {
  c->reset_stats();
  CU(cudaMemsetAsync(c->d_counts, 0, 4 * sizeof(unsigned long long), c->stream));
  Driver d(c, (uint32_t)p, (int)std::min<int64_t>(threshold, INT32_MAX));
  View x{dA, ld, (int)m, (int)n};
  NodeRes res;
  if (iterative) {
    d.threshold = INT32_MAX;  // Algorithm 2 on the whole matrix
    if (m == 0 || n == 0) res = NodeRes{ident(m), ident(n), 0};
    else if (d.fits_small(m, n)) res = d.leaf_small(x);
    else res = d.leaf_global(x);
  } else {
    res = d.rec(x);
  }
  finish_counts(c, d.host_counts, counts);
  for (int64_t i = 0; i < m; ++i) psig[i] = res.P[i];
  for (int64_t j = 0; j < n; ++j) qsig[j] = res.Q[j];
  *rank = res.r;
}

}  // namespace

// =====================================================================================
// C ABI
// =====================================================================================
extern "C" {

int pluq_create(pluq_ctx** out, int device, void* stream) {
  if (!out) return kInvalid;
  pluq_ctx* c = new pluq_ctx();
  c->device = device;
  c->stream = (cudaStream_t)stream;
  int st = guarded(c, [&] {
    CU(cudaMalloc((void**)&c->d_counts, 4 * sizeof(unsigned long long)));
    CU(cudaHostAlloc((void**)&c->h_counts, 4 * sizeof(unsigned long long), cudaHostAllocDefault));
    CU(cudaMalloc((void**)&c->d_flag, sizeof(int)));
    CU(cudaMalloc((void**)&c->d_abort, sizeof(int)));
    CU(cudaHostAlloc((void**)&c->h_flag, sizeof(int), cudaHostAllocDefault));
    CU(cudaMalloc((void**)&c->d_stop, 4 * sizeof(int)));
    CU(cudaHostAlloc((void**)&c->h_stop, 4 * sizeof(int), cudaHostAllocDefault));
    CU(cudaMalloc((void**)&c->d_zflags, pluq_ctx::kMaxDepth * sizeof(int)));
    CU(cudaHostAlloc((void**)&c->h_zflags, pluq_ctx::kMaxDepth * sizeof(int), cudaHostAllocDefault));
    // the context's own pool: freed blocks are kept for reuse between calls (release
    // threshold = max) and trimmed to pool_keep_mb after each API call (guarded); the
    // device's default pool, which other libraries share, is left untouched
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    CU(cudaMemPoolCreate(&c->pool, &props));
    uint64_t thr = ~0ull;
    CU(cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &thr));
    c->tc.pool = c->pool;
    c->ensure_res(1 << 16);
    // rec_smem recurses on the device: give each thread room for the deepest
    // small-node recursion (threshold 1 on a 128x128 node is ~8 frames).
    size_t stack = 0;
    CU(cudaDeviceGetLimit(&stack, cudaLimitStackSize));
    if (stack < 8192) CU(cudaDeviceSetLimit(cudaLimitStackSize, 8192));
  });
  if (st != kOk) {
    *out = nullptr;
    delete c;
    return st;
  }
  *out = c;
  return kOk;
}

int pluq_destroy(pluq_ctx* c) {
  if (!c) return kOk;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  c->tc.release();
  if (c->pin) cudaFreeHost(c->pin);
  if (c->h_bres) cudaFreeHost(c->h_bres);
  if (c->ring) cudaFreeHost(c->ring);
  if (c->node_backup) cudaFree(c->node_backup);
  for (auto e : c->ring_ev) if (e) cudaEventDestroy(e);
  c->hpool.reset();
  for (auto e : c->evpool) cudaEventDestroy(e);
  for (auto s : c->side) if (s) cudaStreamDestroy(s);
  if (c->d_res) cudaFree(c->d_res);
  if (c->h_res) cudaFreeHost(c->h_res);
  if (c->gcount_tab) cudaFree(c->gcount_tab);
  if (c->d_counts) cudaFree(c->d_counts);
  if (c->h_counts) cudaFreeHost(c->h_counts);
  if (c->d_flag) cudaFree(c->d_flag);
  if (c->d_abort) cudaFree(c->d_abort);
  if (c->hi_stream_) cudaStreamDestroy(c->hi_stream_);
  if (c->h_estop) cudaFreeHost(c->h_estop);
  if (c->d_invtab32) cudaFree(c->d_invtab32);
  if (c->d_invtab) cudaFree(c->d_invtab);
  if (c->d_zflags) cudaFree(c->d_zflags);
  if (c->d_stop) cudaFree(c->d_stop);
  if (c->h_stop) cudaFreeHost(c->h_stop);
  if (c->h_zflags) cudaFreeHost(c->h_zflags);
  if (c->h_flag) cudaFreeHost(c->h_flag);
  if (c->pool) {
    cudaDeviceSynchronize();  // stream-ordered frees on the side streams have completed
    cudaMemPoolDestroy(c->pool);
  }
  delete c;
  return kOk;
}

int pluq_release_workspace(pluq_ctx* c) {
  return guarded(c, [&] {
    c->sync();
    if (c->node_backup) CU(cudaFree(c->node_backup));
    c->node_backup = nullptr;
    c->node_backup_bytes = 0;
    if (c->pool) CU(cudaMemPoolTrimTo(c->pool, 0));
  });
}

int pluq_set_stream(pluq_ctx* c, void* stream) {
  if (!c) return kInvalid;
  c->stream = (cudaStream_t)stream;
  return kOk;
}

// Every tuning knob: option name -> context field (pluq_set_option / pluq_get_option).
#define PLUQ_OPTIONS(X)                                                                             \
  X(small_cap, c->small_cap) X(small_threads, c->small_threads) X(batch_threads, c->batch_threads)  \
  X(use_tc, c->use_tc) X(tc_min_dim, c->tc_min_dim) X(tc_min_k, c->tc_min_k)                        \
  X(tc_k_pass, c->tc.k_pass_override) X(tc_cfg, c->tc.variant) X(tc_mnb, c->tc.mn_b)               \
  X(tc_group, c->tc.raster_group) X(tc_cpf, c->tc.c_prefetch) X(tc_grid, c->tc.grid_override)      \
  X(tc_dbg, c->tc.dbg) X(tc_vec, c->tc.vec_limbs) X(tc_pair, c->tc.pair_split) X(tc_time, c->tc.time_mma) X(tc_epi, c->tc.epi_warps)  \
  X(try_generic, c->try_generic) X(time_kernels, c->time_kernels) X(fixed_kernels, c->fixed_kernels) X(batch_dp, c->batch_dp) X(inv32, c->inv32) \
  X(host_chunks, c->host_chunks) X(chunk_shape, c->chunk_shape) X(diag_lazy, c->diag_lazy)          \
  X(lookahead, c->lookahead) X(la_reserve, c->la_reserve) X(exact_kernel, c->exact_kernel)          \
  X(la_pair, c->la_pair) X(la_cap, c->la_cap) X(inner_la, c->inner_la) X(gather_inplace, c->gather_inplace) X(panel_rec, c->panel_rec) X(la_pair_big, c->la_pair_big) X(la_preinv, c->la_preinv) X(la_first_single, c->la_first_single) X(panel_inv, c->panel_inv) X(la_prio, c->la_prio) X(la_side_solve, c->la_side_solve) X(la_adapt, c->la_adapt) X(host_early, c->host_early) X(replay_async, c->replay_async) X(fin_merge, c->fin_merge) X(spec_backup, c->spec_backup) X(spec_unfactor_elems, c->spec_unfactor_elems) X(la_free, c->la_free) X(la_reserve_big, c->la_reserve_big)                             \
  X(rpm_threads, c->rpm_threads) X(rpm_lazy, c->rpm_lazy) X(par_trsm, c->par_trsm)                  \
  X(sym_par, c->sym_par) X(tc_trsm, c->tc_trsm) X(pair_leaves, c->pair_leaves)                      \
  X(stream_fb, c->stream_fb) X(stream_fb_spin, c->stream_fb_spin) X(fb_prefix, c->fb_prefix)        \
  X(rpm_eager, c->rpm_eager) X(tc_trsm_min, c->tc_trsm_min) X(trace_pipeline, c->trace_pipeline)    \
  X(tc_trsm_big, c->tc_trsm_big)                                                                    \
  X(spec_block, c->spec_block) X(spec_check, c->spec_check) X(spec_panel, c->spec_panel)            \
  X(spec_panel_big, c->spec_panel_big) X(spec_big_elems, c->spec_big_elems)                         \
  X(spec_repairs, c->spec_repairs)                                                                  \
  X(check_inputs, c->check_inputs) X(pool_keep_mb, c->pool_keep_mb) X(host_chunk_mb, c->host_chunk_mb)     \
  X(host_wire16, c->host_wire16)                                                                    \
  X(host_threads, c->host_threads)

int pluq_set_option(pluq_ctx* c, const char* key, int64_t value) {
  if (!c || !key) return kInvalid;
  const std::string k(key);
#define PLUQ_SET(name, field)                  \
  if (k == #name) {                            \
    field = (std::decay_t<decltype(field)>)value; \
    return kOk;                                \
  }
  PLUQ_OPTIONS(PLUQ_SET)
#undef PLUQ_SET
  return kInvalid;
}

int pluq_get_option(pluq_ctx* c, const char* key, int64_t* value) {
  if (!c || !key || !value) return kInvalid;
  const std::string k(key);
#define PLUQ_GET(name, field)    \
  if (k == #name) {              \
    *value = (int64_t)(field);   \
    return kOk;                  \
  }
  PLUQ_OPTIONS(PLUQ_GET)
#undef PLUQ_GET
  return kInvalid;
}

const char* pluq_last_error(pluq_ctx* c) { return c ? c->err.c_str() : "null context"; }

int pluq_nonzero(pluq_ctx* c, const uint32_t* dA, int64_t ld, int64_t m, int64_t n, int64_t* out) {
  if (!out || m < 0 || n < 0 || (m > 0 && n > 0 && (!dA || ld < n))) return kInvalid;
  return guarded(c, [&] {
    Ops ops{c, ModP::make(2)};
    *out = (m > 0 && n > 0) ? (ops.nonzero(View{const_cast<uint32_t*>(dA), ld, (int)m, (int)n}) ? 1 : 0) : 0;
  });
}

int pluq_rank_profile_replay(int64_t m, int64_t n, int64_t threshold, int64_t r, const int64_t* prow,
                             const int64_t* pcol, int64_t* p_sigma, int64_t* q_sigma, int64_t* counts) {
  if (m < 0 || n < 0 || m > INT32_MAX / 2 || n > INT32_MAX / 2 || threshold < 1 || r < 0 || r > std::min(m, n))
    return kInvalid;
  if ((r && (!prow || !pcol)) || (m && !p_sigma) || (n && !q_sigma)) return kInvalid;
  try {
    std::vector<int> pr(r), pc(r), seen_r(m, 0), seen_c(n, 0);
    for (int64_t k = 0; k < r; ++k) {
      if (prow[k] < 0 || prow[k] >= m || pcol[k] < 0 || pcol[k] >= n || seen_r[prow[k]]++ || seen_c[pcol[k]]++)
        return kInvalid;  // not a partial permutation
      pr[k] = (int)prow[k];
      pc[k] = (int)pcol[k];
    }
    Perm P, Q;
    Counts cnt{0, 0, 0, 0};
    const int rank = symbolic_replay((int)m, (int)n, (int)std::min<int64_t>(threshold, INT32_MAX), pr, pc, P, Q, cnt);
    if (rank != r) return kInvalid;
    for (int64_t i = 0; i < m; ++i) p_sigma[i] = P[i];
    for (int64_t j = 0; j < n; ++j) q_sigma[j] = Q[j];
    if (counts) {
      counts[0] = (int64_t)cnt.mul; counts[1] = (int64_t)cnt.add; counts[2] = (int64_t)cnt.inv;
      counts[3] = (int64_t)cnt.red;
    }
    return kOk;
  } catch (const std::bad_alloc&) {
    return kNoMemory;
  }
}

int pluq_check_residues(pluq_ctx* c, const uint32_t* dA, int64_t ld, int64_t m, int64_t n, int64_t p) {
  if (int v = validate(m, n, p)) return v;
  if (m > 0 && n > 0 && (!dA || ld < n)) return kInvalid;
  return guarded(c, [&] {
    const int64_t keep = c->check_inputs;
    c->check_inputs = 1;
    try {
      check_residues(c, View{const_cast<uint32_t*>(dA), ld, (int)m, (int)n}, (uint32_t)p);
    } catch (...) {
      c->check_inputs = keep;
      throw;
    }
    c->check_inputs = keep;
  });
}

int pluq_measure_peaks(pluq_ctx* c, double* out, int64_t nout) {
  if (!out || nout < 2) return kInvalid;
  return guarded(c, [&] {
    int dev = 0, sms = 148;
    CU(cudaGetDevice(&dev));
    CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const size_t smem = 1024 + 2 * 128 * 128 + 128 * 128;
    CU(cudaFuncSetAttribute(mma_peak_i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaEvent_t e0, e1;
    CU(cudaEventCreate(&e0));
    CU(cudaEventCreate(&e1));
    const int iters = 4096;
    mma_peak_i8_kernel<<<sms, 128, smem, c->stream>>>(256);  // warm-up
    c->check_launch();
    CU(cudaEventRecord(e0, c->stream));
    mma_peak_i8_kernel<<<sms, 128, smem, c->stream>>>(iters);
    c->check_launch();
    CU(cudaEventRecord(e1, c->stream));
    CU(cudaEventSynchronize(e1));
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, e0, e1));
    out[0] = 2.0 * 128 * 256 * 32 * (double)iters * sms / (ms * 1e-3) / 1e12;  // int8 TOP/s
    double* sink = c->dalloc<double>(256);
    const int fit = 2048;
    mma_peak_f64_kernel<<<sms * 8, 256, 0, c->stream>>>(64, sink);  // warm-up
    c->check_launch();
    CU(cudaEventRecord(e0, c->stream));
    mma_peak_f64_kernel<<<sms * 8, 256, 0, c->stream>>>(fit, sink);
    c->check_launch();
    CU(cudaEventRecord(e1, c->stream));
    CU(cudaEventSynchronize(e1));
    CU(cudaEventElapsedTime(&ms, e0, e1));
    const double mmas = 4.0 * fit * (double)sms * 8 * 8;  // per warp: 4 per iteration; 8 warps per CTA
    out[1] = 2.0 * 8 * 8 * 4 * mmas / (ms * 1e-3) / 1e12;  // fp64 TFLOP/s
    c->dfree(sink);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    c->sync();
  });
}

int pluq_generic_counts(int64_t m, int64_t n, int64_t rank, int64_t threshold, int64_t* counts) {
  if (m < 0 || n < 0 || rank < 0 || rank > std::min(m, n) || threshold < 1 || !counts) return kInvalid;
  Counts c{0, 0, 0, 0};
  generic_counts_rec(m, n, rank, threshold, c);
  counts[0] = (int64_t)c.mul; counts[1] = (int64_t)c.add; counts[2] = (int64_t)c.inv; counts[3] = (int64_t)c.red;
  return kOk;
}

int pluq_last_stats(pluq_ctx* c, int64_t* out, int64_t nout) {
  if (!c || !out) return kInvalid;
  int64_t v[19] = {c->st_launch, c->st_sync, c->st_nodes, c->st_small, c->st_base, c->st_tc, c->st_simt,
                   c->st_zero_skips, c->st_generic, c->st_spec_ok, c->st_spec_fail,
                   (int64_t)(c->t_generic_ms * 1e6f), (int64_t)(c->t_fallback_ms * 1e6f),
                   (int64_t)(c->tc.mma_ms * 1e6f), c->tc.acc_launches, (int64_t)(c->tc.acc_ms * 1e6),
                   (int64_t)c->tc.acc_ops, c->st_repairs, c->st_early_chunks};
  for (int64_t i = 0; i < nout && i < 19; ++i) out[i] = v[i];
  return kOk;
}

int pluq_factor(pluq_ctx* c, uint32_t* dA, int64_t ld, int64_t m, int64_t n, int64_t p,
                int64_t threshold, int64_t* psig, int64_t* qsig, int64_t* rank, int64_t* counts) {
  if (threshold < 1) return kInvalid;
  if (int v = validate(m, n, p)) return v;
  if (ld < n || !rank || (m && !psig) || (n && !qsig)) return kInvalid;
  return guarded(c, [&] {
    // a node that goes straight to the speculative LU validates its entries in the backup
    // copy (one read of the matrix instead of two); every other input is checked here
    const int thr = (int)std::min<int64_t>(threshold, INT32_MAX);
    const bool spec_top = c->try_generic && c->check_inputs && m > 1 && n > 1 && std::min(m, n) > thr &&
                          !(m * n <= c->small_cap && block_smem_bytes(m, n, thr) <= kMaxDynSmem);
    c->range_check_pending = spec_top;
    if (!spec_top) check_residues(c, View{dA, ld, (int)m, (int)n}, (uint32_t)p);
    try {
      factor_device(c, dA, ld, m, n, p, threshold, psig, qsig, rank, counts, false);
    } catch (...) {
      c->range_check_pending = false;
      throw;
    }
    c->range_check_pending = false;
  });
}

int pluq_factor_iterative(pluq_ctx* c, uint32_t* dA, int64_t ld, int64_t m, int64_t n, int64_t p,
                          int64_t* psig, int64_t* qsig, int64_t* rank, int64_t* counts) {
  if (int v = validate(m, n, p)) return v;
  if (ld < n || !rank || (m && !psig) || (n && !qsig)) return kInvalid;
  return guarded(c, [&] {
    check_residues(c, View{dA, ld, (int)m, (int)n}, (uint32_t)p);
    factor_device(c, dA, ld, m, n, p, 1, psig, qsig, rank, counts, true);
  });
}

int64_t pluq_batched_max_elems(pluq_ctx*, int64_t m, int64_t n) {
  return block_smem_bytes(m, n, 30) <= kMaxDynSmem ? m * n : 0;
}

int pluq_factor_batched(pluq_ctx* c, uint32_t* dA, int64_t stride, int64_t batch, int64_t m, int64_t n,
                        int64_t p, int64_t threshold, int32_t* d_p, int32_t* d_q, int32_t* d_rank,
                        uint64_t* d_counts) {
  if (threshold < 1 || batch < 0) return kInvalid;
  if (int v = validate(m, n, p)) return v;
  if (block_smem_bytes(m, n, threshold) > kMaxDynSmem) return kUnsupported;
  if (batch == 0) return kOk;
  if (stride < m * n) return kInvalid;
  return guarded(c, [&] {
    c->reset_stats();
    // canonical-residue check WITHOUT a host round trip before the factorization: the check
    // kernel sets a device flag, every kernel of the batch returns at once when it is set (the
    // input stays untouched), and the host reads the flag once at the end of the call
    const bool check_async = c->check_inputs && m > 0 && n > 0;
    if (check_async) {
      const View xv{dA, stride, (int)batch, (int)(m * n)};
      CU(cudaMemsetAsync(c->d_abort, 0, sizeof(int), c->stream));
      const int n4 = std::max(1, xv.n / 4);
      dim3 rgrid((unsigned)std::min(4, (n4 + 255) / 256), (unsigned)std::min(xv.m, 4096));
      range_check_kernel<<<rgrid, 256, 0, c->stream>>>(xv, (uint32_t)p, c->d_abort);
      c->check_launch();
    }
    SmallArgs a;
    a.batch_dp = (int)c->batch_dp;
    a.abort_flag = check_async ? c->d_abort : nullptr;
    a.a = dA; a.lda = n; a.bstride = stride; a.m = (int)m; a.n = (int)n;
    a.threshold = (int)std::min<int64_t>(threshold, INT32_MAX);
    a.mp = c->modp((uint32_t)p);
    a.p_out = d_p; a.q_out = d_q; a.r_out = d_rank;
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(d_counts);
    if (!cnt) cnt = c->dalloc<unsigned long long>(4 * (size_t)batch);
    a.cnt_out = cnt; a.cnt_accumulate = 0;
    a.invtab = c->invtab((uint32_t)p);
    a.try_generic = (int)c->try_generic;
    a.try_depth = 1;  // depth 0 was attempted by crout_fast_kernel
    a.generic_flag = nullptr;
    unsigned long long* gtab = nullptr;
    if (a.try_generic) gtab = upload_generic_counts(c, m, n, threshold);
    a.generic_counts = gtab;
    int* flags = nullptr;
    a.fail_list = nullptr; a.fail_count = nullptr; a.fail_base = 0;
    if (a.try_generic) {
      // flags: generic flag [batch] | fail count | fail list [batch] | done count | claim
      flags = c->dalloc<int>(2 * (size_t)batch + 3);
      a.generic_flag = flags;
      a.fail_count = flags + batch;
      a.fail_list = flags + batch + 1;
      int* done = flags + 2 * batch + 1;
      int* claim = done + 1;
      const bool streaming = c->stream_fb && c->exact_kernel && batch >= 1024;
      CU(cudaMemsetAsync(a.fail_count, 0, sizeof(int), c->stream));
      uint32_t* prefix = nullptr;
      if (c->fb_prefix && c->exact_kernel && c->fixed_kernels && m == 64 && n == 64 && a.invtab) {
        // the 64x64 generic kernel leaves [t | its Crout image] per failure slot
        a.prefix_slots = (int)std::min<int64_t>(batch, 1024);
        prefix = c->dalloc<uint32_t>((size_t)a.prefix_slots * kPrefixWords);
        a.prefix = prefix;
      }
      if (streaming) {
        CU(cudaMemsetAsync(a.fail_list, 0xff, (size_t)batch * sizeof(int), c->stream));  // -1: slot not ready
        CU(cudaMemsetAsync(done, 0, 2 * sizeof(int), c->stream));
      }
      const size_t cs = crout_smem_bytes(m, n);
      CU(cudaFuncSetAttribute(crout_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cs));
      cudaEvent_t ev[3];
      if (c->time_kernels)
        for (auto& e : ev) { CU(cudaEventCreate(&e)); }
      SmallArgs g = a;
      cudaStream_t cons = c->side_streams()[3];
      cudaEvent_t* sev = c->events(2);
      if (streaming) {
        // a few resident consumer CTAs take the failure list while the generic kernel
        // runs (bounded spin: if they are not co-scheduled they simply give up)
        a.done_count = done;
        a.stream_total = (int)batch;
        g.done_count = done;
        g.stream_total = (int)batch;
        g.claim = claim;
        g.spin_limit = c->stream_fb_spin;
        CU(cudaEventRecord(sev[0], c->stream));
        CU(cudaStreamWaitEvent(cons, sev[0], 0));
      }
      if (c->time_kernels) CU(cudaEventRecord(ev[0], c->stream));
      if (!(c->fixed_kernels && launch_crout_fixed(a, batch, c->stream)))
        crout_fast_kernel<<<(unsigned)batch, (unsigned)c->batch_threads, cs, c->stream>>>(a);
      c->check_launch();
      if (streaming) {
        // submitted AFTER the generic kernel: if the two streams share a hardware queue the
        // consumer simply runs afterwards (it never waits on a kernel that cannot start);
        // otherwise it gets SMs as the generic grid drains
        launch_exact(c, g, (unsigned)c->stream_fb, (unsigned)c->batch_threads, a.fail_list, a.fail_count, cons);
        CU(cudaEventRecord(sev[1], cons));
      }
      if (c->time_kernels) CU(cudaEventRecord(ev[1], c->stream));
      // exact recursion only for the blocks that are not generic (persistent grid); in
      // streaming mode it takes whatever the consumers have not claimed
      const unsigned grid = (unsigned)std::min<int64_t>(batch, 148 * 2);
      launch_exact(c, streaming ? g : a, grid, (unsigned)c->batch_threads, a.fail_list, a.fail_count, c->stream);
      if (streaming) CU(cudaStreamWaitEvent(c->stream, sev[1], 0));
      if (prefix) c->dfree(prefix);
      if (c->time_kernels) {
        CU(cudaEventRecord(ev[2], c->stream));
        CU(cudaEventSynchronize(ev[2]));
        CU(cudaEventElapsedTime(&c->t_generic_ms, ev[0], ev[1]));
        CU(cudaEventElapsedTime(&c->t_fallback_ms, ev[1], ev[2]));
        for (auto& e : ev) cudaEventDestroy(e);
      }
    } else {
      launch_exact(c, a, (unsigned)batch, (unsigned)c->batch_threads, nullptr, nullptr, c->stream);
    }
    if (!d_counts) c->dfree(cnt);
    if (flags) c->dfree(flags);
    if (check_async) {
      CU(cudaMemcpyAsync(c->h_flag, c->d_abort, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      c->sync();
      if (*c->h_flag) throw PluqError(kInvalid, "matrix entries must be canonical residues in [0, p)");
    }
  });
}

// Host dtype <-> uint32 residues on host threads (the reference's storage dtype: float64
// when (p-1)^2 * 8192 <= 2^53, else int64; field.py:75-81).  to_u32 returns false if an entry
// is not a canonical residue (field.py:140-147).
// AVX2 float64 <-> uint32 for the large-matrix pipeline: non-temporal stores into the pinned
// ring and into the caller's float64 buffer (no read-for-ownership of 32 GiB at cfg5).
// Chosen at run time (__builtin_cpu_supports); the scalar loops below are the reference.
__attribute__((target("avx2"))) static bool f64_to_u32_avx2(const double* s, uint32_t* d, int64_t count, uint32_t p) {
  int64_t i = 0;
  bool ok = true;
  const __m256d zero = _mm256_setzero_pd(), pd = _mm256_set1_pd((double)p);
  __m256d bad = _mm256_setzero_pd();
  for (; i < count && (reinterpret_cast<uintptr_t>(d + i) & 15); ++i) {
    const double v = s[i];
    const bool good = v >= 0.0 && v < (double)p && v == std::floor(v);
    d[i] = good ? (uint32_t)v : 0u;
    ok &= good;
  }
  for (; i + 4 <= count; i += 4) {
    const __m256d v = _mm256_loadu_pd(s + i);
    const __m256d fl = _mm256_round_pd(v, _MM_FROUND_TO_NEG_INF | _MM_FROUND_NO_EXC);
    // bad lanes: v < 0, v >= p, v != floor(v), NaN (unordered compares)
    const __m256d b = _mm256_or_pd(_mm256_or_pd(_mm256_cmp_pd(v, zero, _CMP_NGE_UQ), _mm256_cmp_pd(v, pd, _CMP_NLT_UQ)),
                                   _mm256_cmp_pd(v, fl, _CMP_NEQ_UQ));
    bad = _mm256_or_pd(bad, b);
    const __m128i q = _mm256_cvttpd_epi32(_mm256_andnot_pd(b, v));
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + i), q);
  }
  ok &= _mm256_movemask_pd(bad) == 0;
  for (; i < count; ++i) {
    const double v = s[i];
    const bool good = v >= 0.0 && v < (double)p && v == std::floor(v);
    d[i] = good ? (uint32_t)v : 0u;
    ok &= good;
  }
  _mm_sfence();
  return ok;
}
__attribute__((target("avx2"))) static void u32_to_f64_avx2(const uint32_t* s, double* d, int64_t count) {
  int64_t i = 0;
  for (; i < count && (reinterpret_cast<uintptr_t>(d + i) & 31); ++i) d[i] = (double)s[i];
  for (; i + 4 <= count; i += 4)  // residues < 2^31: the signed conversion is exact
    _mm256_stream_pd(d + i, _mm256_cvtepi32_pd(_mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i))));
  for (; i < count; ++i) d[i] = (double)s[i];
  _mm_sfence();
}
// uint16 wire (p <= 2^16): float64 -> uint16 with the same validation, and back.
__attribute__((target("avx2"))) static bool f64_to_u16_avx2(const double* s, uint16_t* d, int64_t count, uint32_t p) {
  int64_t i = 0;
  const __m256d zero = _mm256_setzero_pd(), pd = _mm256_set1_pd((double)p);
  __m256d bad = _mm256_setzero_pd();
  bool ok = true;
  for (; i < count && (reinterpret_cast<uintptr_t>(d + i) & 15); ++i) {
    const double v = s[i];
    const bool good = v >= 0.0 && v < (double)p && v == std::floor(v);
    d[i] = good ? (uint16_t)v : 0;
    ok &= good;
  }
  for (; i + 8 <= count; i += 8) {
    __m128i q[2];
    for (int h = 0; h < 2; ++h) {
      const __m256d v = _mm256_loadu_pd(s + i + 4 * h);
      const __m256d fl = _mm256_round_pd(v, _MM_FROUND_TO_NEG_INF | _MM_FROUND_NO_EXC);
      const __m256d b = _mm256_or_pd(_mm256_or_pd(_mm256_cmp_pd(v, zero, _CMP_NGE_UQ), _mm256_cmp_pd(v, pd, _CMP_NLT_UQ)),
                                     _mm256_cmp_pd(v, fl, _CMP_NEQ_UQ));
      bad = _mm256_or_pd(bad, b);
      q[h] = _mm256_cvttpd_epi32(_mm256_andnot_pd(b, v));
    }
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + i), _mm_packus_epi32(q[0], q[1]));
  }
  ok &= _mm256_movemask_pd(bad) == 0;
  for (; i < count; ++i) {
    const double v = s[i];
    const bool good = v >= 0.0 && v < (double)p && v == std::floor(v);
    d[i] = good ? (uint16_t)v : 0;
    ok &= good;
  }
  _mm_sfence();
  return ok;
}
__attribute__((target("avx2"))) static void u16_to_f64_avx2(const uint16_t* s, double* d, int64_t count) {
  int64_t i = 0;
  for (; i < count && (reinterpret_cast<uintptr_t>(d + i) & 31); ++i) d[i] = (double)s[i];
  for (; i + 4 <= count; i += 4)
    _mm256_stream_pd(d + i, _mm256_cvtepi32_pd(_mm_cvtepu16_epi32(_mm_loadl_epi64(reinterpret_cast<const __m128i*>(s + i)))));
  for (; i < count; ++i) d[i] = (double)s[i];
  _mm_sfence();
}

static bool have_avx2() {
  static const bool v = __builtin_cpu_supports("avx2");
  return v;
}

static bool host_to_u32(const void* src, bool is_f64, uint32_t* dst, int64_t count, uint32_t p) {
  if (is_f64 && have_avx2()) return f64_to_u32_avx2(static_cast<const double*>(src), dst, count, p);
  bool ok = true;
  if (is_f64) {
    const double* s = static_cast<const double*>(src);
    for (int64_t i = 0; i < count; ++i) {
      const double v = s[i];
      const bool good = v >= 0.0 && v < (double)p && v == std::floor(v);
      dst[i] = good ? (uint32_t)v : 0u;
      ok &= good;
    }
  } else {
    const int64_t* s = static_cast<const int64_t*>(src);
    for (int64_t i = 0; i < count; ++i) {
      const int64_t v = s[i];
      const bool good = v >= 0 && v < (int64_t)p;
      dst[i] = good ? (uint32_t)v : 0u;
      ok &= good;
    }
  }
  return ok;
}
static bool host_to_u16(const void* src, bool is_f64, uint16_t* dst, int64_t count, uint32_t p) {
  if (is_f64 && have_avx2()) return f64_to_u16_avx2(static_cast<const double*>(src), dst, count, p);
  bool ok = true;
  for (int64_t i = 0; i < count; ++i) {
    bool good;
    uint32_t v;
    if (is_f64) {
      const double x = static_cast<const double*>(src)[i];
      good = x >= 0.0 && x < (double)p && x == std::floor(x);
      v = good ? (uint32_t)x : 0u;
    } else {
      const int64_t x = static_cast<const int64_t*>(src)[i];
      good = x >= 0 && x < (int64_t)p;
      v = good ? (uint32_t)x : 0u;
    }
    dst[i] = (uint16_t)v;
    ok &= good;
  }
  return ok;
}
static void host_from_u16(const uint16_t* src, bool is_f64, void* dst, int64_t count) {
  if (is_f64 && have_avx2()) return u16_to_f64_avx2(src, static_cast<double*>(dst), count);
  for (int64_t i = 0; i < count; ++i) {
    if (is_f64) static_cast<double*>(dst)[i] = (double)src[i];
    else static_cast<int64_t*>(dst)[i] = (int64_t)src[i];
  }
}

static void host_from_u32(const uint32_t* src, bool is_f64, void* dst, int64_t count) {
  if (is_f64 && have_avx2()) return u32_to_f64_avx2(src, static_cast<double*>(dst), count);
  if (is_f64) {
    double* d = static_cast<double*>(dst);
    for (int64_t i = 0; i < count; ++i) d[i] = (double)src[i];
  } else {
    int64_t* d = static_cast<int64_t*>(dst);
    for (int64_t i = 0; i < count; ++i) d[i] = (int64_t)src[i];
  }
}

static int factor_host(pluq_ctx* c, void* hA, bool is_f64, int64_t m, int64_t n, int64_t p, int64_t threshold,
                       int64_t* psig, int64_t* qsig, int64_t* rank, int64_t* counts) {
  if (threshold < 1) return kInvalid;
  if (int v = validate(m, n, p)) return v;
  if (!rank || (m && !psig) || (n && !qsig)) return kInvalid;
  return guarded(c, [&] {
    const int64_t cnt = m * n;
    const size_t chunk = (size_t)std::max<int64_t>(1, c->host_chunk_mb) << 20;  // bytes of uint32 per chunk
    if ((size_t)cnt * 4 <= chunk) {
      // small matrix: one pageable copy in the host dtype, converted on the device
      void* raw = c->dalloc<char>((size_t)cnt * 8);
      uint32_t* dA = c->dalloc<uint32_t>((size_t)cnt);
      if (cnt) CU(cudaMemcpyAsync(raw, hA, (size_t)cnt * 8, cudaMemcpyHostToDevice, c->stream));
      int grid = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 16, (cnt + 255) / 256));
      if (cnt) {
        CU(cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
        if (is_f64) from_f64_kernel<<<grid, 256, 0, c->stream>>>((const double*)raw, dA, cnt, (uint32_t)p, c->d_flag);
        else from_i64_kernel<<<grid, 256, 0, c->stream>>>((const int64_t*)raw, dA, cnt, (uint32_t)p, c->d_flag);
        c->check_launch();
        CU(cudaMemcpyAsync(c->h_flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        if (*c->h_flag) {  // nothing was modified: the host buffer is only written at the end
          c->dfree(dA);
          c->dfree(raw);
          throw PluqError(kInvalid, "matrix entries must be canonical residues in [0, p)");
        }
      }
      factor_device(c, dA, n, m, n, p, threshold, psig, qsig, rank, counts, false);
      if (cnt) {
        if (is_f64) to_f64_kernel<<<grid, 256, 0, c->stream>>>(dA, (double*)raw, cnt);
        else to_i64_kernel<<<grid, 256, 0, c->stream>>>(dA, (int64_t*)raw, cnt);
        c->check_launch();
        CU(cudaMemcpyAsync(hA, raw, (size_t)cnt * 8, cudaMemcpyDeviceToHost, c->stream));
      }
      c->dfree(dA);
      c->dfree(raw);
      c->sync();
      return;
    }
    // Large matrix: a chunked pipeline through a pinned ring.  Host threads convert the
    // caller's float64/int64 rows to uint32 residues (checking them) while the previous
    // chunks are in flight, so PCIe carries 4 bytes per entry instead of 8; on the way back
    // D2H of later chunks overlaps the widening of earlier ones.  The caller's buffer is
    // written only after the factorization, so invalid input leaves it untouched.
    // p <= 2^16: the wire carries uint16 (2 bytes per entry), widened on the device
    const bool w16 = p <= 65536 && c->host_wire16;
    const size_t wb = w16 ? 2 : 4;                                 // wire bytes per entry
    const size_t ce = chunk / wb;                                  // entries per chunk
    const int64_t nch = (cnt + (int64_t)ce - 1) / (int64_t)ce;
    char* ring = c->staging_ring(chunk);
    HostPool& hp = c->host_pool();
    const int parts = hp.size() * 2;
    uint32_t* dA = c->dalloc<uint32_t>((size_t)cnt);
    uint16_t* dstage = w16 ? c->dalloc<uint16_t>((size_t)pluq_ctx::kRing * ce) : nullptr;
    auto wgrid = [](int64_t ne) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>(148 * 8, (ne / 8 + 255) / 256)); };
    cudaStream_t* ss = c->side_streams();
    cudaStream_t sin = ss[0], sout = ss[1];
    cudaEvent_t* ev = c->ring_ev;
    cudaEvent_t* je = c->events(2);
    CU(cudaEventRecord(je[0], c->stream));  // dA's allocation is ordered before the copies
    CU(cudaStreamWaitEvent(sin, je[0], 0));
    const size_t esz = 8;  // float64 and int64 alike
    std::atomic<bool> ok{true};
    for (int64_t k = 0; k < nch; ++k) {
      const int s = (int)(k % pluq_ctx::kRing);
      if (k >= pluq_ctx::kRing) CU(cudaEventSynchronize(ev[s]));  // the slot's previous copy is done
      const int64_t e0 = k * (int64_t)ce, ne = std::min<int64_t>((int64_t)ce, cnt - e0);
      uint32_t* slot = reinterpret_cast<uint32_t*>(ring + (size_t)s * chunk);
      uint16_t* slot16 = reinterpret_cast<uint16_t*>(ring + (size_t)s * chunk);
      const char* src = static_cast<const char*>(hA) + (size_t)e0 * esz;
      hp.run(parts, [&](int t) {  // per-thread ranges start on 16-entry boundaries
        const int64_t a = t ? (ne * t / parts) & ~int64_t(15) : 0;
        const int64_t b = t + 1 < parts ? (ne * (t + 1) / parts) & ~int64_t(15) : ne;
        if (b > a && !(w16 ? host_to_u16(src + (size_t)a * esz, is_f64, slot16 + a, b - a, (uint32_t)p)
                           : host_to_u32(src + (size_t)a * esz, is_f64, slot + a, b - a, (uint32_t)p)))
          ok.store(false);
      });
      if (w16) {  // the slot's event then covers both the pinned and the device staging slot
        CU(cudaMemcpyAsync(dstage + (size_t)s * ce, slot16, (size_t)ne * 2, cudaMemcpyHostToDevice, sin));
        widen16_kernel<<<wgrid(ne), 256, 0, sin>>>(dstage + (size_t)s * ce, dA + e0, ne);
        c->check_launch();
      } else {
        CU(cudaMemcpyAsync(dA + e0, slot, (size_t)ne * 4, cudaMemcpyHostToDevice, sin));
      }
      CU(cudaEventRecord(ev[s], sin));
    }
    CU(cudaEventRecord(je[1], sin));
    CU(cudaStreamWaitEvent(c->stream, je[1], 0));
    if (!ok.load()) {
      c->dfree(dA);
      if (dstage) c->dfree(dstage);
      c->sync();
      throw PluqError(kInvalid, "matrix entries must be canonical residues in [0, p)");
    }
    auto issue = [&](int64_t k) {
      const int s = (int)(k % pluq_ctx::kRing);
      const int64_t e0 = k * (int64_t)ce, ne = std::min<int64_t>((int64_t)ce, cnt - e0);
      if (w16) {
        narrow16_kernel<<<wgrid(ne), 256, 0, sout>>>(dA + e0, dstage + (size_t)s * ce, ne);
        {  // not c->check_launch(): this lambda also runs on the early-download thread (no shared counters)
          const cudaError_t le = cudaGetLastError();
          if (le != cudaSuccess) throw PluqError(kCuda, std::string("kernel launch: ") + cudaGetErrorString(le));
        }
        CU(cudaMemcpyAsync(ring + (size_t)s * chunk, dstage + (size_t)s * ce, (size_t)ne * 2, cudaMemcpyDeviceToHost, sout));
      } else {
        CU(cudaMemcpyAsync(ring + (size_t)s * chunk, dA + e0, (size_t)ne * 4, cudaMemcpyDeviceToHost, sout));
      }
      CU(cudaEventRecord(ev[s], sout));
    };
    auto widen = [&](int64_t k) {  // chunk k has arrived in its ring slot: widen it into the caller's buffer
      const int s = (int)(k % pluq_ctx::kRing);
      const int64_t e0 = k * (int64_t)ce, ne = std::min<int64_t>((int64_t)ce, cnt - e0);
      const uint32_t* slot = reinterpret_cast<const uint32_t*>(ring + (size_t)s * chunk);
      const uint16_t* slot16 = reinterpret_cast<const uint16_t*>(ring + (size_t)s * chunk);
      char* dst = static_cast<char*>(hA) + (size_t)e0 * esz;
      hp.run(parts, [&](int t) {
        const int64_t a = t ? (ne * t / parts) & ~int64_t(15) : 0;
        const int64_t b = t + 1 < parts ? (ne * (t + 1) / parts) & ~int64_t(15) : ne;
        if (b <= a) return;
        if (w16) host_from_u16(slot16 + a, is_f64, dst + (size_t)a * esz, b - a);
        else host_from_u32(slot + a, is_f64, dst + (size_t)a * esz, b - a);
      });
    };
    // Early download (option host_early): while the speculative LU of the root still runs, a
    // second host thread copies back and widens every chunk whose rows it has announced final
    // (Driver::early_publish); the caller's buffer was validated during the upload, so writing
    // results into it early is safe.  Pivot repairs rotate a few columns in ALL rows: those
    // columns are fetched again at the end; a failed speculation invalidates the early chunks.
    int64_t kdone = 0;
    std::thread dl;
    std::atomic<bool> fin{false};
    std::exception_ptr dl_err;
    const bool early = c->host_early != 0 && nch > 2 * pluq_ctx::kRing;
    if (early) {
      c->early_rows.store(0);
      c->early_invalid.store(false);
      c->early_patches.clear();
      const int want = 4096;
      if (c->h_estop_cap < want) {
        if (c->h_estop) CU(cudaFreeHost(c->h_estop));
        CU(cudaHostAlloc((void**)&c->h_estop, want * sizeof(int), cudaHostAllocDefault));
        c->h_estop_cap = want;
      }
      c->h_estop_n = 0;
      c->early_on = true;
      dl = std::thread([&] {
        try {
          CU(cudaSetDevice(c->device));
          auto final_chunk = [&](int64_t k) {  // every row of chunk k announced final
            if (k >= nch) return false;
            const int64_t e_end = std::min<int64_t>((k + 1) * (int64_t)ce, cnt);
            return (e_end - 1) / n < c->early_rows.load();
          };
          int64_t issued = 0;
          while (!fin.load()) {
            if (c->early_invalid.load()) break;
            while (issued < kdone + pluq_ctx::kRing - 1 && final_chunk(issued)) issue(issued++);
            if (kdone < issued) {
              CU(cudaEventSynchronize(ev[kdone % pluq_ctx::kRing]));
              widen(kdone);
              ++kdone;
            } else {
              std::this_thread::sleep_for(std::chrono::microseconds(200));
            }
          }
          for (; kdone < issued; ++kdone) {  // drain what was issued
            CU(cudaEventSynchronize(ev[kdone % pluq_ctx::kRing]));
            widen(kdone);
          }
        } catch (...) {
          dl_err = std::current_exception();
        }
      });
    }
    try {
      factor_device(c, dA, n, m, n, p, threshold, psig, qsig, rank, counts, false);
    } catch (...) {
      fin.store(true);
      if (dl.joinable()) dl.join();
      c->early_on = false;
      throw;
    }
    fin.store(true);
    if (dl.joinable()) dl.join();
    c->early_on = false;
    if (dl_err) std::rethrow_exception(dl_err);
    if (early && c->early_invalid.load()) kdone = 0;
    c->st_early_chunks = kdone;
    CU(cudaEventRecord(je[0], c->stream));
    CU(cudaStreamWaitEvent(sout, je[0], 0));
    const int64_t k_first = kdone;
    for (int64_t k = k_first; k < std::min<int64_t>(nch, k_first + pluq_ctx::kRing); ++k) issue(k);
    for (int64_t k = k_first; k < nch; ++k) {
      CU(cudaEventSynchronize(ev[k % pluq_ctx::kRing]));
      widen(k);
      if (k + pluq_ctx::kRing < nch) issue(k + pluq_ctx::kRing);
    }
    if (early && k_first > 0) {
      // columns rotated by pivot repairs after some of their rows had been downloaded
      const int64_t rows_early = std::min<int64_t>(m, (k_first * (int64_t)ce + n - 1) / n);
      for (const auto& pr : c->early_patches) {
        const int64_t pr_rows = std::min<int64_t>(pr.first, rows_early), c0 = pr.first, w = pr.second + 1;
        if (pr_rows <= 0) continue;
        std::vector<uint32_t> tmp((size_t)pr_rows * w);
        CU(cudaMemcpy2DAsync(tmp.data(), (size_t)w * 4, dA + c0, (size_t)n * 4, (size_t)w * 4, (size_t)pr_rows,
                             cudaMemcpyDeviceToHost, sout));
        CU(cudaStreamSynchronize(sout));
        for (int64_t i = 0; i < pr_rows; ++i)
          for (int64_t j = 0; j < w; ++j) {
            const size_t e = (size_t)i * n + c0 + j;
            if (is_f64) static_cast<double*>(hA)[e] = (double)tmp[(size_t)i * w + j];
            else static_cast<int64_t*>(hA)[e] = (int64_t)tmp[(size_t)i * w + j];
          }
      }
    }
    CU(cudaEventRecord(je[1], sout));
    CU(cudaStreamWaitEvent(c->stream, je[1], 0));
    c->dfree(dA);
    if (dstage) c->dfree(dstage);
    c->sync();
  });
}

int pluq_factor_host_f64(pluq_ctx* c, double* hA, int64_t m, int64_t n, int64_t p, int64_t threshold,
                         int64_t* psig, int64_t* qsig, int64_t* rank, int64_t* counts) {
  return factor_host(c, hA, true, m, n, p, threshold, psig, qsig, rank, counts);
}

int pluq_factor_host_i64(pluq_ctx* c, int64_t* hA, int64_t m, int64_t n, int64_t p, int64_t threshold,
                         int64_t* psig, int64_t* qsig, int64_t* rank, int64_t* counts) {
  return factor_host(c, hA, false, m, n, p, threshold, psig, qsig, rank, counts);
}

int pluq_factor_batched_host_f64(pluq_ctx* c, double* hA, int64_t batch, int64_t m, int64_t n, int64_t p,
                                 int64_t threshold, int64_t* psig, int64_t* qsig, int64_t* ranks) {
  if (threshold < 1 || batch < 0) return kInvalid;
  if (int v = validate(m, n, p)) return v;
  if (block_smem_bytes(m, n, threshold) > kMaxDynSmem) return kUnsupported;
  const auto hentry = std::chrono::steady_clock::now();
  return guarded(c, [&] {
    const int64_t mn = m * n;
    if (batch == 0 || mn == 0) {
      for (int64_t b = 0; b < batch; ++b) {
        for (int64_t i = 0; i < m; ++i) psig[b * m + i] = i;
        for (int64_t j = 0; j < n; ++j) qsig[b * n + j] = j;
        ranks[b] = 0;
      }
      return;
    }
    // Chunked pipeline on four streams: H2D of chunk k+1 (sin), the generic kernel of
    // chunk k (compute), the exact recursion over chunk k's few non-generic blocks plus
    // the f64 conversion (sfb: a handful of CTAs, latency-bound, so it overlaps the next
    // chunk's generic kernel), and D2H of chunk k-1 (sout).
    const int64_t nchunks = std::max<int64_t>(1, std::min<int64_t>(c->host_chunks, batch));
    // tent-shaped chunk sizes (weights min(k+1, C-k)): the D2H stream is the bottleneck
    // once it runs, so the first chunk is small (D2H starts early) and so is the last
    // (its compute and D2H follow the final H2D)
    std::vector<int64_t> cb0(nchunks + 1, 0);
    {
      const int64_t C = nchunks;
      int64_t wsum = 0;
      auto wt = [&](int64_t kk) { return c->chunk_shape ? std::min(kk + 1, C - kk) : int64_t(1); };
      for (int64_t kk = 0; kk < C; ++kk) wsum += wt(kk);
      int64_t acc = 0, wacc = 0;
      for (int64_t kk = 0; kk < C; ++kk) {
        wacc += wt(kk);
        const int64_t end = kk == C - 1 ? batch : std::max(acc, batch * wacc / wsum);
        cb0[kk] = acc;
        acc = end;
      }
      cb0[C] = batch;
    }
    double* raw = c->dalloc<double>((size_t)batch * mn);
    uint32_t* dA = c->dalloc<uint32_t>((size_t)batch * mn);
    int32_t* dp = c->dalloc<int32_t>((size_t)(batch * (m + n + 1)));
    CU(cudaStreamSynchronize(c->stream));  // allocations visible to the side streams
    // the exact kernel of a chunk is a few latency-bound CTAs: round-robin them over
    // several streams so that the fallbacks of consecutive chunks overlap
    constexpr int kFb = 4;
    cudaStream_t* ss = c->side_streams();
    cudaStream_t sin = ss[0], sout = ss[1], *sfbs = ss + 2;
    const bool tr = c->trace_pipeline != 0;
    // events: in / generic / done / out per chunk, + start/end (timing-enabled when tracing)
    std::vector<cudaEvent_t> tev;
    cudaEvent_t* evs;
    if (tr) {
      tev.resize(5 * nchunks + 2);
      for (auto& e : tev) CU(cudaEventCreate(&e));
      evs = tev.data();
    } else {
      evs = c->events(5 * nchunks + 2);
    }
    cudaEvent_t *ev_in = evs, *ev_gen = evs + nchunks, *ev_done = evs + 2 * nchunks, *ev_out = evs + 3 * nchunks;
    cudaEvent_t *ev_res = evs + 4 * nchunks;
    cudaEvent_t ev0 = evs[5 * nchunks], ev_end = evs[5 * nchunks + 1];
    // per-block results (P, Q, rank) come back per chunk into pinned memory and are
    // widened to the caller's int64 arrays while later chunks are still in flight
    int32_t* host = c->batch_results((size_t)(batch * (m + n + 1)));
    const auto h0 = std::chrono::steady_clock::now();
    const ModP mp = c->modp((uint32_t)p);
    SmallArgs a;
    a.batch_dp = (int)c->batch_dp;
    a.lda = n; a.bstride = mn; a.m = (int)m; a.n = (int)n;
    a.threshold = (int)std::min<int64_t>(threshold, INT32_MAX);
    a.mp = mp; a.invtab = c->invtab((uint32_t)p);
    a.try_generic = (int)c->try_generic;
    a.try_depth = 1;
    a.generic_flag = nullptr;
    unsigned long long* gtab = a.try_generic ? upload_generic_counts(c, m, n, threshold) : nullptr;
    a.generic_counts = gtab;
    unsigned long long* cnt = c->dalloc<unsigned long long>(4 * (size_t)batch);
    a.cnt_accumulate = 0;
    const size_t cs = crout_smem_bytes(m, n);
    CU(cudaFuncSetAttribute(crout_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cs));
    // flags: per-block generic flag [batch] | per-chunk failure count [nchunks] | failure
    // list [batch] (chunk k lists its failures, as global indices, from slot cb0[k] on)
    int* flags = a.try_generic ? c->dalloc<int>(2 * (size_t)batch + nchunks) : nullptr;
    a.fail_list = nullptr; a.fail_count = nullptr; a.fail_base = 0;
    if (flags) CU(cudaMemsetAsync(flags + batch, 0, sizeof(int) * nchunks, c->stream));
    CU(cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
    CU(cudaStreamSynchronize(c->stream));
    CU(cudaEventRecord(ev0, sin));
    int64_t last = 0;
    for (int64_t k = 0; k < nchunks; ++k) {
      const int64_t b0 = cb0[k], nb = cb0[k + 1] - cb0[k];
      if (nb <= 0) continue;
      last = k;
      CU(cudaMemcpyAsync(raw + b0 * mn, hA + b0 * mn, (size_t)nb * mn * 8, cudaMemcpyHostToDevice, sin));
      CU(cudaEventRecord(ev_in[k], sin));
      CU(cudaStreamWaitEvent(c->stream, ev_in[k], 0));
      const int64_t cntk = nb * mn;
      const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 16, (cntk + 255) / 256));
      from_f64_kernel<<<grid, 256, 0, c->stream>>>(raw + b0 * mn, dA + b0 * mn, cntk, (uint32_t)p, c->d_flag);
      c->check_launch();
      // chunk k's results are one contiguous record [P (nb x m) | Q (nb x n) | rank (nb)]
      // so that a single D2H copy returns them
      int32_t* rec = dp + b0 * (m + n + 1);
      a.a = dA + b0 * mn;
      a.p_out = rec; a.q_out = rec + nb * m; a.r_out = rec + nb * (m + n);
      a.cnt_out = cnt + 4 * b0;
      cudaStream_t tail = c->stream;
      if (flags) {
        a.generic_flag = flags + b0;
        a.fail_base = 0;  // chunk-local indices
        a.fail_count = flags + batch + k;
        a.fail_list = flags + batch + nchunks + b0;
        if (!(c->fixed_kernels && launch_crout_fixed(a, nb, c->stream)))
          crout_fast_kernel<<<(unsigned)nb, (unsigned)c->batch_threads, cs, c->stream>>>(a);
        c->check_launch();
        CU(cudaEventRecord(ev_gen[k], c->stream));
        cudaStream_t sfb = sfbs[k % kFb];
        CU(cudaStreamWaitEvent(sfb, ev_gen[k], 0));
        SmallArgs g = a;
        g.generic_flag = nullptr;
        launch_exact(c, g, (unsigned)std::min<int64_t>(nb, 148 * 2), (unsigned)c->batch_threads, a.fail_list,
                     a.fail_count, sfb);
        tail = sfb;
      } else {
        launch_exact(c, a, (unsigned)nb, (unsigned)c->batch_threads, nullptr, nullptr, c->stream);
      }
      to_f64_kernel<<<grid, 256, 0, tail>>>(dA + b0 * mn, raw + b0 * mn, cntk);
      c->check_launch();
      CU(cudaEventRecord(ev_done[k], tail));
      CU(cudaStreamWaitEvent(sout, ev_done[k], 0));
      CU(cudaMemcpyAsync(hA + b0 * mn, raw + b0 * mn, (size_t)nb * mn * 8, cudaMemcpyDeviceToHost, sout));
      CU(cudaEventRecord(ev_out[k], sout));
      CU(cudaMemcpyAsync(host + b0 * (m + n + 1), rec, (size_t)nb * (m + n + 1) * 4, cudaMemcpyDeviceToHost, sout));
      CU(cudaEventRecord(ev_res[k], sout));
    }
    CU(cudaEventRecord(ev_end, sout));
    for (int64_t k = 0; k <= last; ++k) {
      CU(cudaEventSynchronize(ev_res[k]));
      const int64_t b0 = cb0[k], nb = cb0[k + 1] - cb0[k];
      const int32_t* hr = host + b0 * (m + n + 1);
      for (int64_t i = 0; i < nb * m; ++i) psig[b0 * m + i] = hr[i];
      for (int64_t i = 0; i < nb * n; ++i) qsig[b0 * n + i] = hr[nb * m + i];
      for (int64_t i = 0; i < nb; ++i) ranks[b0 + i] = hr[nb * (m + n) + i];
    }
    CU(cudaStreamSynchronize(sout));
    CU(cudaStreamSynchronize(c->stream));
    for (int q = 0; q < kFb; ++q) CU(cudaStreamSynchronize(sfbs[q]));
    const auto h1 = std::chrono::steady_clock::now();
    if (tr) {
      auto ms = [&](cudaEvent_t e) { float v = 0.f; cudaEventElapsedTime(&v, ev0, e); return v; };
      fprintf(stderr, "pipeline: setup %.3f ms, enqueue+wait %.3f ms, device end %.3f ms\n",
              std::chrono::duration<double, std::milli>(h0 - hentry).count(),
              std::chrono::duration<double, std::milli>(h1 - h0).count(), ms(ev_end));
      for (int64_t k = 0; k <= last; ++k)
        fprintf(stderr, "  chunk %lld: h2d %.3f gen %.3f done %.3f d2h %.3f\n", (long long)k, ms(ev_in[k]),
                ms(ev_gen[k]), ms(ev_done[k]), ms(ev_out[k]));
      for (auto e : tev) cudaEventDestroy(e);
    }
    c->dfree(cnt);
    if (flags) c->dfree(flags);
    c->dfree(dp);
    c->dfree(dA);
    c->dfree(raw);  // stream-ordered: every stream that used these buffers has been synchronised
    // non-canonical entries (flagged by the conversions): ValueError like the reference's
    // DenseMatrix construction; blocks holding them were factored as if they were 0
    CU(cudaMemcpyAsync(c->h_flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    if (*c->h_flag) throw PluqError(kInvalid, "matrix entries must be canonical residues in [0, p)");
    if (tr)
      fprintf(stderr, "pipeline: frees %.3f ms\n",
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h1).count());
  });
}

int pluq_modgemm_sub(pluq_ctx* c, uint32_t* dC, int64_t ldc, const uint32_t* dA, int64_t lda,
                     const uint32_t* dB, int64_t ldb, int64_t m, int64_t n, int64_t k, int64_t p) {
  if (int v = validate(m, n, p)) return v;
  if (k < 0 || k > INT32_MAX / 2) return kInvalid;
  return guarded(c, [&] {
    Ops ops{c, c->modp((uint32_t)p)};
    ops.gemm(View{dC, ldc, (int)m, (int)n}, View{const_cast<uint32_t*>(dA), lda, (int)m, (int)k},
             View{const_cast<uint32_t*>(dB), ldb, (int)k, (int)n});
  });
}

int pluq_modgemm_sub_tc(pluq_ctx* c, uint32_t* dC, int64_t ldc, const uint32_t* dA, int64_t lda,
                        const uint32_t* dB, int64_t ldb, int64_t m, int64_t n, int64_t k, int64_t p) {
  if (int v = validate(m, n, p)) return v;
  if (k < 0 || k > INT32_MAX / 2) return kInvalid;
  if (!c) return kInvalid;
  int st = kOk;
  int g = guarded(c, [&] {
    st = c->tc.run(View{dC, ldc, (int)m, (int)n}, View{const_cast<uint32_t*>(dA), lda, (int)m, (int)k},
                   View{const_cast<uint32_t*>(dB), ldb, (int)k, (int)n}, ModP::make((uint32_t)p), c->stream);
    if (st != kOk && st != kUnsupported) throw PluqError(st, c->tc.last_error);
  });
  return g != kOk ? g : st;
}

int pluq_trsm_llu(pluq_ctx* c, const uint32_t* dL, int64_t ldl, uint32_t* dB, int64_t ldb, int64_t r,
                  int64_t n, int64_t p) {
  if (int v = validate(r, n, p)) return v;
  return guarded(c, [&] {
    Ops ops{c, c->modp((uint32_t)p)};
    ops.trsm_l(View{const_cast<uint32_t*>(dL), ldl, (int)r, (int)r}, View{dB, ldb, (int)r, (int)n});
  });
}

int pluq_trsm_ru(pluq_ctx* c, uint32_t* dB, int64_t ldb, const uint32_t* dU, int64_t ldu, int64_t m,
                 int64_t r, int64_t p) {
  if (int v = validate(m, r, p)) return v;
  int zero = 0;
  int g = guarded(c, [&] {
    View u{const_cast<uint32_t*>(dU), ldu, (int)r, (int)r};
    if (r > 0) {
      CU(cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
      diag_zero_kernel<<<(unsigned)((r + 255) / 256), 256, 0, c->stream>>>(u, c->d_flag);
      c->check_launch();
      CU(cudaMemcpyAsync(c->h_flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      c->sync();
      if (*c->h_flag) { zero = 1; return; }
    }
    Ops ops{c, c->modp((uint32_t)p)};
    ops.trsm_u(View{dB, ldb, (int)m, (int)r}, u);
  });
  if (g != kOk) return g;
  if (zero) { c->err = "upper triangular factor has a zero diagonal entry"; return kZeroDivision; }
  return kOk;
}

int pluq_permute_rows(pluq_ctx* c, uint32_t* dX, int64_t ld, int64_t rows, int64_t cols, const int64_t* g) {
  if (rows < 0 || cols < 0 || (rows && !g)) return kInvalid;
  return guarded(c, [&] {
    Perm gg(rows);
    for (int64_t i = 0; i < rows; ++i) gg[i] = (int32_t)g[i];
    Ops ops{c, ModP::make(2)};
    ops.gather_rows(View{dX, ld, (int)rows, (int)cols}, gg);
  });
}

int pluq_permute_cols(pluq_ctx* c, uint32_t* dX, int64_t ld, int64_t rows, int64_t cols, const int64_t* g) {
  if (rows < 0 || cols < 0 || (cols && !g)) return kInvalid;
  return guarded(c, [&] {
    Perm gg(cols);
    for (int64_t j = 0; j < cols; ++j) gg[j] = (int32_t)g[j];
    Ops ops{c, ModP::make(2)};
    ops.gather_cols(View{dX, ld, (int)rows, (int)cols}, gg);
  });
}

}  // extern "C"
