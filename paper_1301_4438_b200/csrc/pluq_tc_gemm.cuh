// Tensor-core modular GEMM  C <- C - A B  (mod p)  on sm_100a.
//
// Replaces ClassicalKernels.mm_acc (/root/reference/pkg/src/pluq/kernels.py:38-55),
// whose arithmetic core is numpy float64/int64 matmul (field.py:149-161).
//
// Representation: residues (< p < 2^31) are split into L = ceil(bits(p-1)/8)
// unsigned 8-bit limbs.  A B = sum_{i,j} 2^{8(i+j)} A_i B_j, so the L^2 limb
// products are accumulated by `tcgen05.mma.cta_group::1.kind::i8` (u8 x u8 -> s32)
// into 2L-1 TMEM accumulators, one per limb position s = i+j.  Position s holds at
// most L products of K terms each < 255^2, so one pass is exact while
// K * L * 255^2 < 2^31; longer K is split into passes.  The fused epilogue reads
// the accumulators with tcgen05.ld, recombines them by Horner mod p
// (v <- v*256 + acc_s), subtracts from C and stores.
//
// Data movement: a conversion kernel writes the limb planes of the A view
// (row-major = K-major) and of B^T (K-major) into zero-padded scratch, so every
// TMA box is in bounds and no K tail needs masking.  TMA (SWIZZLE_128B) stages
// 128x128-byte A tiles and BNx128-byte B tiles per limb into a STAGES-deep
// mbarrier ring; one elected thread issues the MMAs; four epilogue warps own the
// 128 TMEM lanes.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "pluq_common.cuh"

namespace pluq {

// ------------------------------- PTX wrappers ---------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tmem_alloc(uint32_t* holder, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(holder)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void mma_i8(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// K-major, SWIZZLE_128B shared-memory matrix descriptor (8-row groups 1024 B apart).
__device__ __forceinline__ uint64_t desc_k_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;              // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;    // stride byte offset
  d |= (uint64_t)1 << 46;              // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;              // SWIZZLE_128B
  return d;
}

// MN-major, SWIZZLE_128B descriptor for a tile whose MN extent is one 128-byte swizzle
// atom (rows = K, 128 bytes of N each): 8-row K groups 1024 B apart (SBO); LBO (the
// stride between MN atoms) is unused with a single atom.
__device__ __forceinline__ uint64_t desc_mn_sw128(uint32_t saddr, uint32_t lbo = 128 * 128) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;  // leading byte offset: next 128-byte MN atom
  d |= (uint64_t)(1024 >> 4) << 32;          // stride byte offset: next group of 8 K rows
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// kind::i8 instruction descriptor: s32 accumulate, u8 x u8, A K-major, B K-major
// (mnb = false) or MN-major (mnb = true, bit 16), M=128.
__host__ __device__ constexpr uint32_t idesc_i8(int n, bool mnb = false) {
  return (2u << 4) | (0u << 7) | (0u << 10) | ((mnb ? 1u : 0u) << 16) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(128 >> 4) << 24);
}

// Persistent tiling: each CTA (one per SM) walks output tiles; TMEM holds TWO
// accumulator sets (NPOS positions x BN columns each) so the epilogue of tile t
// overlaps the MMAs of tile t+1.
// V = 0: narrow tiles, two TMEM accumulator sets (epilogue overlapped with the next
// tile's MMAs).  V = 1: wide tiles with ONE accumulator set: the operand bytes per MAC
// drop from (BM+BN)/(L*BM*BN) = 0.0117 (L=2, BN=64) to 0.0078 (BN=128), which is what
// the L2->SM bandwidth (~6.3 KB/cycle chip-wide) allows at >60 % of the int8 MMA rate;
// the unoverlapped epilogue costs ~1/(K/32) of a K=4096 tile.
template <int L, int V>
struct TcCfg;
template <> struct TcCfg<1, 0> { static constexpr int BN = 256, STAGES = 4, NBUF = 2; };
template <> struct TcCfg<2, 0> { static constexpr int BN = 64, STAGES = 4, NBUF = 2; };
template <> struct TcCfg<3, 0> { static constexpr int BN = 32, STAGES = 3, NBUF = 2; };
template <> struct TcCfg<4, 0> { static constexpr int BN = 32, STAGES = 2, NBUF = 2; };
template <> struct TcCfg<1, 1> { static constexpr int BN = 256, STAGES = 4, NBUF = 2; };
template <> struct TcCfg<2, 1> { static constexpr int BN = 128, STAGES = 3, NBUF = 1; };
template <> struct TcCfg<3, 1> { static constexpr int BN = 96, STAGES = 2, NBUF = 1; };
template <> struct TcCfg<4, 1> { static constexpr int BN = 64, STAGES = 2, NBUF = 1; };
// V = 2 (two-limb primes, MN-major B): two passes per tile, see tc_modgemm2p_kernel.
template <> struct TcCfg<2, 2> { static constexpr int BN = 128, STAGES = 4, NBUF = 1; };

constexpr int TC_BM = 128, TC_BK = 128;

// Epilogue: EPI warps (8 or 16; 4 per TMEM lane quarter), each draining BN / (EPI / 4)
// columns of its 32 rows in chunks of CW columns (16 with 8 warps, 8 with 16 warps).
template <int EPI>
struct TcEpi {
  static constexpr int CW = EPI == 16 ? 8 : 16;
  static constexpr size_t SMEM = (size_t)EPI * 32 * (CW + 1) * 4;  // per-warp transpose tile
  static constexpr int THREADS = (4 + EPI) * 32;                   // warps 0 TMA, 1 MMA, 2 TMEM alloc, 3 idle
};

template <int L, int V, int EPI = 8>
constexpr size_t tc_smem_bytes() {
  // V = 2 stages hold ONE A limb tile and both B limb tiles
  return 1024 + (size_t)TcCfg<L, V>::STAGES * ((V == 2 ? 1 : L) * TC_BM * TC_BK + L * TcCfg<L, V>::BN * TC_BK) + 256 +
         TcEpi<EPI>::SMEM;
}

template <int CW>
__device__ __forceinline__ void tmem_ld_cw(uint32_t taddr, uint32_t (&v)[CW]) {
  if constexpr (CW == 16) tmem_ld16(taddr, v);
  else tmem_ld8(taddr, v);
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// MNB: B limb planes are row-major k x n (MN-major operand, written by the same
// vectorised split as A, no transpose pass); requires BN == 128 (one swizzle atom).
template <int L, int V, bool MNB, int EPI>
__global__ void __launch_bounds__(TcEpi<EPI>::THREADS, 1)
    tc_modgemm_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, View c,
                      int m_pad, int n_pad, int kblocks, ModP mp, const int* stop, int dbg, int group,
                      int c_prefetch) {
  const int kplane = kblocks * TC_BK;  // rows of one MN-major B limb plane
  if (stop && *reinterpret_cast<const volatile int*>(stop)) return;
  constexpr int BN = TcCfg<L, V>::BN, STAGES = TcCfg<L, V>::STAGES, NBUF = TcCfg<L, V>::NBUF;
  static_assert(!MNB || BN == 128, "MN-major B needs one 128-byte swizzle atom per tile");
  constexpr int NPOS = 2 * L - 1;
  // MNB (L = 2): the two B limb tiles sit side by side along N in shared memory, so each
  // A limb multiplies [B_lo | B_hi] in ONE N = 256 MMA (2 MMAs per K step, not 4).  The
  // A_hi MMA is aimed one position to the right of the A_lo one, so the two middle products
  // A_lo B_hi and A_hi B_lo accumulate into the SAME TMEM columns: the set is
  // [P0 | P1 | P2] = [A_lo B_lo | A_lo B_hi + A_hi B_lo | A_hi B_hi], 3 x 128 columns (P1 <
  // K * 2 * 255^2 < 2^31 is the one-pass bound k_pass already enforces).  Only the tile's
  // first K step differs (P2 must start from zero while P1 accumulates): A_hi [B_lo|B_hi]
  // initialises [P1 | P2], then A_lo B_lo initialises P0 and A_lo B_hi adds into P1.
  constexpr bool CAT = MNB && L == 2;
  constexpr int ACC_COLS = NPOS * BN;  // one accumulator set
  constexpr uint32_t TCOLS = 512;
  static_assert(NBUF * ACC_COLS <= 512, "the accumulator sets must fit in TMEM");
  constexpr uint32_t A_TILE = TC_BM * TC_BK, B_TILE = BN * TC_BK;
  constexpr uint32_t STAGE_BYTES = L * (A_TILE + B_TILE);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                                  // [STAGES][L][128x128]
  uint8_t* sB = smem + (size_t)STAGES * L * A_TILE;    // [STAGES][L][BNx128]
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + (size_t)STAGES * L * B_TILE);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // [NBUF]
  uint64_t* tempty = tfull + NBUF;    // [NBUF]
  uint32_t* tholder = reinterpret_cast<uint32_t*>(tempty + NBUF);
  uint32_t* epi_smem = reinterpret_cast<uint32_t*>(sB + (size_t)STAGES * L * B_TILE + 256);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_n = n_pad / BN, tiles_m = m_pad / TC_BM, tiles = tiles_m * tiles_n;
  // grouped rasterisation: consecutive tiles walk `group` tile rows before moving to the
  // next tile column, so a wave of persistent CTAs touches a compact set of A row panels
  // and B column panels (they stay in L2 instead of streaming B once per wave)
  auto tile_coords = [&](int tile, int& m0, int& n0) {
    const int g = group > 0 ? group : tiles_m;
    const int span = g * tiles_n, gid = tile / span, fm = gid * g, gsz = min(tiles_m - fm, g);
    const int rem = tile - gid * span;
    m0 = (fm + rem % gsz) * TC_BM;
    n0 = (rem / gsz) * BN;
  };

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < NBUF; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], EPI); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) tmem_alloc(tholder, TCOLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tholder;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    uint32_t g = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
      int m0, n0;
      tile_coords(tile, m0, n0);
      for (int kb = 0; kb < kblocks; ++kb, ++g) {
        const uint32_t s = g % STAGES;
        mbar_wait(&empty[s], ((g / STAGES) & 1) ^ 1);
        if ((dbg & 1) && g >= (uint32_t)STAGES) {  // diagnostics: MMA rate without operand traffic
          mbar_arrive(&full[s]);
          continue;
        }
        mbar_expect_tx(&full[s], STAGE_BYTES);
#pragma unroll
        for (int l = 0; l < L; ++l) {
          tma_load_2d(sA + ((size_t)s * L + l) * A_TILE, &ta, &full[s], kb * TC_BK, l * m_pad + m0);
          if (MNB)
            tma_load_2d(sB + ((size_t)s * L + l) * B_TILE, &tb, &full[s], n0, l * kplane + kb * TC_BK);
          else
            tma_load_2d(sB + ((size_t)s * L + l) * B_TILE, &tb, &full[s], kb * TC_BK, l * n_pad + n0);
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer (single thread) ----------------
    constexpr uint32_t idesc = idesc_i8(BN, MNB);
    constexpr uint32_t idesc_cat = idesc_i8(2 * BN, true);
    uint32_t g = 0, local = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++local) {
      const uint32_t buf = local % NBUF, use = local / NBUF;
      mbar_wait(&tempty[buf], (use & 1) ^ 1);
      tc_fence_after();
      const uint32_t dacc = tbase + buf * ACC_COLS;
      for (int kb = 0; kb < kblocks; ++kb, ++g) {
        const uint32_t s = g % STAGES;
        mbar_wait(&full[s], (g / STAGES) & 1);
        tc_fence_after();
        const uint32_t a0 = smem_u32(sA + (size_t)s * L * A_TILE);
        const uint32_t b0 = smem_u32(sB + (size_t)s * L * B_TILE);
        if constexpr (CAT) {
          // the A_lo MMAs of the stage first, then the A_hi ones: an MMA whose columns only
          // partly overlap the previous one's (offset by one position) waits for it, so the
          // stage has two such switches instead of eight (tools/gemm_dbg.py)
#pragma unroll
          for (int kk = 0; kk < TC_BK / 32; ++kk) {
            const uint64_t bd = desc_mn_sw128(b0 + kk * 32 * 128, B_TILE);
            const uint64_t alo = desc_k_sw128(a0 + kk * 32);
            if (kb == 0 && kk == 0) {
              mma_i8(dacc + (uint32_t)BN, desc_k_sw128(a0 + A_TILE), bd, idesc_cat, 0u);  // [P1|P2] = A_hi [B_lo|B_hi]
              mma_i8(dacc, alo, bd, idesc, 0u);                                          //  P0     = A_lo B_lo
              mma_i8(dacc + (uint32_t)BN, alo, desc_mn_sw128(b0 + B_TILE, B_TILE), idesc, 1u);  // P1 += A_lo B_hi
            } else {
              mma_i8(dacc, alo, bd, idesc_cat, 1u);  // [P0 | P1] += A_lo [B_lo | B_hi]
            }
          }
#pragma unroll
          for (int kk = (kb == 0 ? 1 : 0); kk < TC_BK / 32; ++kk)  // [P1 | P2] += A_hi [B_lo | B_hi]
            mma_i8(dacc + (uint32_t)BN, desc_k_sw128(a0 + A_TILE + kk * 32),
                   desc_mn_sw128(b0 + kk * 32 * 128, B_TILE), idesc_cat, 1u);
          mma_commit(&empty[s]);
          continue;
        }
#pragma unroll
        for (int kk = 0; kk < TC_BK / 32; ++kk) {
#pragma unroll
          for (int i = 0; i < L; ++i) {
#pragma unroll
            for (int j = 0; j < L; ++j) {
              const int pos = i + j;
              const int first_i = pos < L ? 0 : pos - (L - 1);
              const uint32_t acc = (kb > 0 || kk > 0 || i != first_i) ? 1u : 0u;
              const uint64_t ad = desc_k_sw128(a0 + i * A_TILE + kk * 32);
              const uint64_t bd = MNB ? desc_mn_sw128(b0 + j * B_TILE + kk * 32 * 128)
                                      : desc_k_sw128(b0 + j * B_TILE + kk * 32);
              mma_i8(dacc + (uint32_t)(pos * BN), ad, bd, idesc, acc);
            }
          }
        }
        mma_commit(&empty[s]);
      }
      mma_commit(&tfull[buf]);
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: TMEM -> recombine mod p -> C ----------------
    // 8 warps: TMEM sub-partition q = warp % 4 (lanes 32q..32q+31 = tile rows), column
    // half h.  Per 16-column chunk a thread holds its row; the limb positions are
    // combined exactly in 64 bits (sum acc_s * 2^(8s) < 2^64 for L <= 3 since every
    // acc_s < 2^31; L = 4 reduces after position 4) and reduced ONCE, then the 32 x 16
    // values are transposed through shared memory so that the read-modify-write of C is
    // coalesced (lanes along a row, 16 independent loads in flight per thread).
    constexpr int TC_CW = TcEpi<EPI>::CW, RSTEP = 32 / TC_CW;
    const int q = warp & 3, h = (warp - 4) >> 2;
    constexpr int HALF = BN / (EPI / 4);  // columns of this warp's share
    static_assert(HALF % TC_CW == 0, "epilogue chunking");
    uint32_t* tr = epi_smem + (warp - 4) * 32 * (TC_CW + 1);
    const int tc_col = lane % TC_CW, tc_row0 = lane / TC_CW;  // transposed phase: RSTEP rows x CW columns
    // limb positions of one 16-column chunk -> 16 reduced values of this thread's row
    auto combine = [&](uint32_t lane_base, int cc, uint32_t (&v)[TC_CW]) {
      uint32_t acc[NPOS][TC_CW];
#pragma unroll
      for (int s = 0; s < NPOS; ++s) tmem_ld_cw<TC_CW>(lane_base + (uint32_t)(s * BN + cc), acc[s]);
      tmem_ld_wait();
#pragma unroll
      for (int t = 0; t < TC_CW; ++t) {
        if (NPOS <= 5) {
          uint64_t x = 0;
#pragma unroll
          for (int s = 0; s < NPOS; ++s) x += (uint64_t)acc[s][t] << (8 * s);
          v[t] = reduce64(x, mp);
        } else {
          uint64_t hi = 0;
#pragma unroll
          for (int s = 4; s < NPOS; ++s) hi += (uint64_t)acc[s][t] << (8 * (s - 4));
          uint64_t x = (uint64_t)reduce64(hi, mp) << 32;
#pragma unroll
          for (int s = 0; s < 4; ++s) x += (uint64_t)acc[s][t] << (8 * s);
          v[t] = reduce64(x, mp);
        }
      }
    };
    // transpose a chunk through shared memory and apply C <- C - v, coalesced
    auto apply = [&](int m0, int n0, int cc, const uint32_t (&v)[TC_CW]) {
#pragma unroll
      for (int t = 0; t < TC_CW; ++t) tr[lane * (TC_CW + 1) + t] = v[t];
      __syncwarp();
      const int col = n0 + cc + tc_col;
      uint32_t w[TC_CW], cur[TC_CW];
#pragma unroll
      for (int kk = 0; kk < TC_CW; ++kk) {
        const int rr = tc_row0 + RSTEP * kk, row = m0 + q * 32 + rr;
        w[kk] = tr[rr * (TC_CW + 1) + tc_col];
        cur[kk] = (row < c.m && col < c.n) ? c.row(row)[col] : 0u;
      }
#pragma unroll
      for (int kk = 0; kk < TC_CW; ++kk) {
        const int row = m0 + q * 32 + tc_row0 + RSTEP * kk;
        if (row < c.m && col < c.n) c.row(row)[col] = submod(cur[kk], w[kk], mp);
      }
      __syncwarp();  // tr is reused by the next chunk
    };
    constexpr int NCH = HALF / TC_CW;
    uint32_t local = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++local) {
      const uint32_t buf = local % NBUF, use = local / NBUF;
      int m0, n0;
      tile_coords(tile, m0, n0);
      if (c_prefetch) {
        // pull this thread's C row segment (HALF columns) into L2 while the tile's MMAs
        // run, so the read-modify-write after the TMEM drain hits L2 instead of HBM
        const int row = m0 + q * 32 + lane, col = n0 + h * HALF;
        if (row < c.m && col < c.n) {
          const char* p = reinterpret_cast<const char*>(c.row(row) + col);
          const int bytes = min(HALF, c.n - col) * 4;
          for (int o = 0; o < bytes; o += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(p + o));
        }
      }
      mbar_wait(&tfull[buf], use & 1);
      tc_fence_after();
      if (dbg & 2) {  // diagnostics: MMA + operand feed rate without the epilogue
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
        continue;
      }
      const uint32_t lane_base = tbase + buf * ACC_COLS + ((uint32_t)(q * 32) << 16);
      if constexpr (CAT && NBUF == 1 && NCH <= 4) {
        // (tools/gemm_ab.py: +18 % at 16384^2 x 1024, but 2-3 % SLOWER on the power-capped far
        // updates of cfg5, so only outputs up to 2^28 entries take it; dbg 8 / 16 force off / on)
        const bool fast40 = mp.mu32 != 0u && mp.p >= 512u && !(dbg & 8) &&
                            ((dbg & 16) || (long long)c.m * c.n <= (1ll << 28));
        const uint32_t e32f = fast40 ? (uint32_t)((1ull << 32) % mp.p) : 0u;
        const uint32_t mu40f = fast40 ? (uint32_t)((1ull << 40) / mp.p) : 0u, np40 = 0u - mp.p;
        // two limbs, single accumulator set: the critical section (TMEM busy, tensor pipe
        // idle) holds only the drain and the exact 48-bit recombination, two IMAD.WIDE per
        // value: x = P0 + 2^8 P1 + 2^16 P2 < 2^31 (1 + 2^8 + 2^16).  TMEM is released
        // before the Barrett reductions and the C read-modify-write.
        uint64_t xv[NCH][TC_CW];
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          uint32_t p0[TC_CW], p1[TC_CW], p2[TC_CW];
          const uint32_t cc = (uint32_t)(h * HALF + ch * TC_CW);
          tmem_ld_cw<TC_CW>(lane_base + cc, p0);
          tmem_ld_cw<TC_CW>(lane_base + (uint32_t)BN + cc, p1);
          tmem_ld_cw<TC_CW>(lane_base + (uint32_t)(2 * BN) + cc, p2);
          tmem_ld_wait();
#pragma unroll
          for (int t = 0; t < TC_CW; ++t)
            xv[ch][t] = (uint64_t)p0[t] + (uint64_t)p1[t] * 256u + (uint64_t)p2[t] * 65536u;
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
        if (dbg & 4) continue;  // diagnostics: no C read-modify-write
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          uint32_t v[TC_CW];
          if (fast40) {
            // p < 2^16: fold the high word (x < 2^47: hi < 2^15) with 2^32 mod p, then the
            // 5-instruction reduction of pluq_diag2.cuh (7 instructions instead of ~18)
#pragma unroll
            for (int t = 0; t < TC_CW; ++t) {
              const uint64_t y = (uint64_t)(uint32_t)(xv[ch][t] >> 32) * e32f + (uint32_t)xv[ch][t];
              v[t] = red40(y, mp.p, np40, mu40f);
            }
          } else {
#pragma unroll
            for (int t = 0; t < TC_CW; ++t) v[t] = reduce64(xv[ch][t], mp);
          }
          apply(m0, n0, h * HALF + ch * TC_CW, v);
        }
      } else if constexpr (NBUF == 1 && NCH <= 4) {
        // single accumulator set: drain TMEM into registers first and release it, so the
        // next tile's MMAs overlap this tile's C read-modify-write
        uint32_t v[NCH][TC_CW];
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) combine(lane_base, h * HALF + ch * TC_CW, v[ch]);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
        if (dbg & 4) continue;  // diagnostics: no C read-modify-write
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) apply(m0, n0, h * HALF + ch * TC_CW, v[ch]);
      } else {
#pragma unroll 1
        for (int cc = h * HALF; cc < (h + 1) * HALF; cc += TC_CW) {
          uint32_t v[TC_CW];
          combine(lane_base, cc, v);
          apply(m0, n0, cc, v);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tbase, TCOLS);
  }
}

// Two-pass variant for two-limb primes (p < 2^16) with MN-major B: each 128 x 128 tile is
// computed as pass X = A_lo [B_lo | B_hi] (TMEM columns 0..255: X0 | X1) and then pass
// Y = A_hi [B_lo | B_hi] (columns 256..511: Y0 | Y1), each over the whole K range, with its
// own full/empty accumulator barriers.  The epilogue drains X0 + 2^8 X1 as soon as pass X
// is done (while pass Y runs) and 2^8 Y0 + 2^16 Y1 after pass Y (while the next tile's
// pass X runs), so the tensor pipe never waits for a TMEM drain: the one-set kernel
// loses the whole drain (256 KB of TMEM at 64 B/cycle) plus the MMA-drain round trip per
// tile, ~40 % at K = 2048 (tools/gemm_dbg.py).  Price: B is loaded once per pass (+50 %
// operand bytes).  The pass-X partial stays in registers until pass Y is drained, so C is
// read-modified-written once per tile.
__global__ void __launch_bounds__(TcEpi<8>::THREADS, 1)
    tc_modgemm2p_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, View c,
                        int m_pad, int n_pad, int kblocks, ModP mp, const int* stop, int dbg, int group,
                        int c_prefetch) {
  constexpr int L = 2, BN = 128, STAGES = TcCfg<2, 2>::STAGES, EPI = 8;
  const int kplane = kblocks * TC_BK;
  if (stop && *reinterpret_cast<const volatile int*>(stop)) return;
  constexpr uint32_t TCOLS = 512;
  constexpr uint32_t A_TILE = TC_BM * TC_BK, B_TILE = BN * TC_BK;
  constexpr uint32_t STAGE_BYTES = A_TILE + L * B_TILE;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                                  // [STAGES][128x128]
  uint8_t* sB = smem + (size_t)STAGES * A_TILE;        // [STAGES][L][BNx128]
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + (size_t)STAGES * L * B_TILE);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // [2]: pass X, pass Y accumulators ready
  uint64_t* tempty = tfull + 2;       // [2]: pass X, pass Y columns drained
  uint32_t* tholder = reinterpret_cast<uint32_t*>(tempty + 2);
  uint32_t* epi_smem = reinterpret_cast<uint32_t*>(sB + (size_t)STAGES * L * B_TILE + 256);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_n = n_pad / BN, tiles_m = m_pad / TC_BM, tiles = tiles_m * tiles_n;
  auto tile_coords = [&](int tile, int& m0, int& n0) {
    const int g = group > 0 ? group : tiles_m;
    const int span = g * tiles_n, gid = tile / span, fm = gid * g, gsz = min(tiles_m - fm, g);
    const int rem = tile - gid * span;
    m0 = (fm + rem % gsz) * TC_BM;
    n0 = (rem / gsz) * BN;
  };
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], EPI); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) tmem_alloc(tholder, TCOLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tholder;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer: per tile, pass X (A_lo) then pass Y (A_hi) ----------
    uint32_t g = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
      int m0, n0;
      tile_coords(tile, m0, n0);
      for (int pass = 0; pass < 2; ++pass)
        for (int kb = 0; kb < kblocks; ++kb, ++g) {
          const uint32_t s = g % STAGES;
          mbar_wait(&empty[s], ((g / STAGES) & 1) ^ 1);
          if ((dbg & 1) && g >= (uint32_t)STAGES) {
            mbar_arrive(&full[s]);
            continue;
          }
          mbar_expect_tx(&full[s], STAGE_BYTES);
          tma_load_2d(sA + (size_t)s * A_TILE, &ta, &full[s], kb * TC_BK, pass * m_pad + m0);
#pragma unroll
          for (int l = 0; l < L; ++l)
            tma_load_2d(sB + ((size_t)s * L + l) * B_TILE, &tb, &full[s], n0, l * kplane + kb * TC_BK);
        }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer: N = 256 MMAs against [B_lo | B_hi] --------------------
    constexpr uint32_t idesc_cat = idesc_i8(2 * BN, true);
    uint32_t g = 0, local = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++local) {
      for (int pass = 0; pass < 2; ++pass) {
        mbar_wait(&tempty[pass], (local & 1) ^ 1);
        tc_fence_after();
        const uint32_t dacc = tbase + (uint32_t)(pass * 2 * BN);
        for (int kb = 0; kb < kblocks; ++kb, ++g) {
          const uint32_t s = g % STAGES;
          mbar_wait(&full[s], (g / STAGES) & 1);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + (size_t)s * A_TILE);
          const uint32_t b0 = smem_u32(sB + (size_t)s * L * B_TILE);
#pragma unroll
          for (int kk = 0; kk < TC_BK / 32; ++kk)
            mma_i8(dacc, desc_k_sw128(a0 + kk * 32), desc_mn_sw128(b0 + kk * 32 * 128, B_TILE), idesc_cat,
                   (kb > 0 || kk > 0) ? 1u : 0u);
          mma_commit(&empty[s]);
        }
        mma_commit(&tfull[pass]);
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: per pass, TMEM -> partial value mod p -> C -= value -----
    constexpr int TC_CW = TcEpi<EPI>::CW, RSTEP = 32 / TC_CW, HALF = BN / 2, NCH = HALF / TC_CW;
    const int q = warp & 3, h = (warp - 4) >> 2;
    uint32_t* tr = epi_smem + (warp - 4) * 32 * (TC_CW + 1);
    const int tc_col = lane % TC_CW, tc_row0 = lane / TC_CW;
    auto apply = [&](int m0, int n0, int cc, const uint32_t (&v)[TC_CW]) {
#pragma unroll
      for (int t = 0; t < TC_CW; ++t) tr[lane * (TC_CW + 1) + t] = v[t];
      __syncwarp();
      const int col = n0 + cc + tc_col;
      uint32_t w[TC_CW], cur[TC_CW];
#pragma unroll
      for (int kk = 0; kk < TC_CW; ++kk) {
        const int rr = tc_row0 + RSTEP * kk, row = m0 + q * 32 + rr;
        w[kk] = tr[rr * (TC_CW + 1) + tc_col];
        cur[kk] = (row < c.m && col < c.n) ? c.row(row)[col] : 0u;
      }
#pragma unroll
      for (int kk = 0; kk < TC_CW; ++kk) {
        const int row = m0 + q * 32 + tc_row0 + RSTEP * kk;
        if (row < c.m && col < c.n) c.row(row)[col] = submod(cur[kk], w[kk], mp);
      }
      __syncwarp();
    };
    uint32_t local = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++local) {
      int m0, n0;
      tile_coords(tile, m0, n0);
      if (c_prefetch) {
        const int row = m0 + q * 32 + lane, col = n0 + h * HALF;
        if (row < c.m && col < c.n) {
          const char* p = reinterpret_cast<const char*>(c.row(row) + col);
          const int bytes = min(HALF, c.n - col) * 4;
          for (int o = 0; o < bytes; o += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(p + o));
        }
      }
      // pass X: v = X0 + 2^8 X1 (mod p) into registers, release the X columns; pass Y:
      // v += 2^8 Y0 + 2^16 Y1 (mod p), release the Y columns; then ONE C read-modify-write
      // (every accumulator < 2^31, so each partial fits 48 bits before its reduction)
      uint32_t v[NCH][TC_CW];
      for (int pass = 0; pass < 2; ++pass) {
        mbar_wait(&tfull[pass], local & 1);
        tc_fence_after();
        if (dbg & 2) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[pass]);
          continue;
        }
        const uint32_t lane_base = tbase + (uint32_t)(pass * 2 * BN) + ((uint32_t)(q * 32) << 16);
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          const int cc = h * HALF + ch * TC_CW;
          uint32_t lo[TC_CW], hi[TC_CW];
          tmem_ld_cw<TC_CW>(lane_base + (uint32_t)cc, lo);
          tmem_ld_cw<TC_CW>(lane_base + (uint32_t)(BN + cc), hi);
          tmem_ld_wait();
#pragma unroll
          for (int t = 0; t < TC_CW; ++t) {
            const uint32_t part = reduce64(((uint64_t)lo[t] + ((uint64_t)hi[t] << 8)) << (8 * pass), mp);
            v[ch][t] = pass ? addmod(v[ch][t], part, mp) : part;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[pass]);
      }
      if (dbg & 6) continue;  // diagnostics: 4 = no C read-modify-write
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) apply(m0, n0, h * HALF + ch * TC_CW, v[ch]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tbase, TCOLS);
  }
}

// Limb planes of a row-major view (K-major operand): out[l][i][kk] = limb_l(v[i][kk]),
// zero-padded to rows_pad x k_pad.  4 consecutive bytes per thread.
__global__ void limb_rows_kernel(View v, uint8_t* out, int L, int rows_pad, int k_pad, const int* stop) {
  if (stop && *reinterpret_cast<const volatile int*>(stop)) return;
  const int64_t plane = (int64_t)rows_pad * k_pad;
  const int kq = k_pad / 4;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)rows_pad * kq;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t / kq), k4 = (int)(t - (int64_t)i * kq) * 4;
    uint32_t w[4] = {0, 0, 0, 0};
    if (i < v.m) {
      const uint32_t* r = v.row(i);
#pragma unroll
      for (int e = 0; e < 4; ++e) w[e] = (k4 + e < v.n) ? r[k4 + e] : 0u;
    }
    for (int l = 0; l < L; ++l) {
      const int sh = 8 * l;
      uint32_t packed = ((w[0] >> sh) & 255u) | (((w[1] >> sh) & 255u) << 8) | (((w[2] >> sh) & 255u) << 16) |
                        (((w[3] >> sh) & 255u) << 24);
      *reinterpret_cast<uint32_t*>(out + l * plane + (int64_t)i * k_pad + k4) = packed;
    }
  }
}

// Limb planes of B^T (B is k x n row-major): out[l][j][kk] = limb_l(B[kk][j]),
// zero-padded to n_pad x k_pad; 32x32 tiles transposed through shared memory.
__global__ void limb_cols_kernel(View b, uint8_t* out, int L, int n_pad, int k_pad, const int* stop) {
  if (stop && *reinterpret_cast<const volatile int*>(stop)) return;
  __shared__ uint32_t tile[32][33];
  const int64_t plane = (int64_t)n_pad * k_pad;
  const int j0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 256 threads: 8 rows per pass
  for (int r = ty; r < 32; r += 8) {
    const int kk = k0 + r, j = j0 + tx;
    tile[r][tx] = (kk < b.m && j < b.n) ? b.at(kk, j) : 0u;
  }
  __syncthreads();
  // each thread writes 4 consecutive kk bytes of one column j
  const int jj = threadIdx.x >> 3, kq = (threadIdx.x & 7) * 4;
  if (j0 + jj < n_pad) {
    for (int l = 0; l < L; ++l) {
      const int sh = 8 * l;
      uint32_t packed = ((tile[kq][jj] >> sh) & 255u) | (((tile[kq + 1][jj] >> sh) & 255u) << 8) |
                        (((tile[kq + 2][jj] >> sh) & 255u) << 16) | (((tile[kq + 3][jj] >> sh) & 255u) << 24);
      *reinterpret_cast<uint32_t*>(out + l * plane + (int64_t)(j0 + jj) * k_pad + k0 + kq) = packed;
    }
  }
}

// Vectorised limb split of a row-major view: 16 consecutive k per thread, one 16-byte
// store per limb plane (k_pad is a multiple of 128, so every store is aligned).
__device__ __forceinline__ void limb_rows16_body(const View& v, uint8_t* out, int L, int rows_pad, int k_pad) {
  const int64_t plane = (int64_t)rows_pad * k_pad;
  const int kq = k_pad / 16;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)rows_pad * kq;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t / kq), k16 = (int)(t - (int64_t)i * kq) * 16;
    uint32_t w[16];
    if (i < v.m) {
      const uint32_t* r = v.row(i) + k16;
      if (k16 + 16 <= v.n && (reinterpret_cast<uintptr_t>(r) & 15) == 0) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint4 q = reinterpret_cast<const uint4*>(r)[e];
          w[4 * e] = q.x; w[4 * e + 1] = q.y; w[4 * e + 2] = q.z; w[4 * e + 3] = q.w;
        }
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) w[e] = (k16 + e < v.n) ? r[e] : 0u;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 16; ++e) w[e] = 0u;
    }
    for (int l = 0; l < L; ++l) {
      const int sh = 8 * l;
      uint32_t pk[4];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        pk[e] = ((w[4 * e] >> sh) & 255u) | (((w[4 * e + 1] >> sh) & 255u) << 8) |
                (((w[4 * e + 2] >> sh) & 255u) << 16) | (((w[4 * e + 3] >> sh) & 255u) << 24);
      *reinterpret_cast<uint4*>(out + l * plane + (int64_t)i * k_pad + k16) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
  }
}

__global__ void limb_rows16_kernel(View v, uint8_t* out, int L, int rows_pad, int k_pad, const int* stop) {
  if (stop && *reinterpret_cast<const volatile int*>(stop)) return;
  limb_rows16_body(v, out, L, rows_pad, k_pad);
}
// Both operands of one GEMM call in ONE launch (blockIdx.y selects the operand): the small
// GEMMs of the panel chain pay one launch latency less per call.
__global__ void limb_rows16_pair_kernel(View va, uint8_t* outa, int rows_a, int k_a, View vb, uint8_t* outb, int rows_b,
                                        int k_b, int L, const int* stop) {
  if (stop && *reinterpret_cast<const volatile int*>(stop)) return;
  if (blockIdx.y == 0) limb_rows16_body(va, outa, L, rows_a, k_a);
  else limb_rows16_body(vb, outb, L, rows_b, k_b);
}

// ------------------------- peak microbenchmarks -------------------------
// int8 tensor-core peak: one elected thread per CTA issues `iters` back-to-back
// tcgen05.mma.kind::i8 128x256x32 (SS operands, 32 KB of shared memory, contents
// irrelevant) into one TMEM accumulator; one CTA per SM.  ops = 2*128*256*32 per MMA.
__global__ void __launch_bounds__(128, 1) mma_peak_i8_kernel(int iters) {
  extern __shared__ __align__(1024) uint8_t smem_pk[];
  __shared__ uint64_t done;
  __shared__ uint32_t holder;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_pk) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(&holder, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = holder;
  if (threadIdx.x == 32) {
    constexpr uint32_t idesc = idesc_i8(256);
    const uint64_t ad = desc_k_sw128(smem_u32(base));
    const uint64_t bd = desc_k_sw128(smem_u32(base + 128 * 128));
    for (int i = 0; i < iters; ++i) mma_i8(t, ad, bd, idesc, i > 0 ? 1u : 0u);
    mma_commit(&done);
    mbar_wait(&done, 0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(t, 256);
  }
}

// FP64 DMMA peak (mma.sync m8n8k4): every warp runs `iters` dependent-free groups of 4
// independent MMAs; flops = 2*8*8*4 per MMA.
__global__ void __launch_bounds__(256) mma_peak_f64_kernel(int iters, double* sink) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c0[2] = {0, 0}, c1[2] = {0, 0}, c2[2] = {0, 0}, c3[2] = {0, 0};
  for (int i = 0; i < iters; ++i) {
#define PLUQ_DMMA(c)                                                                                      \
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"            \
               : "+d"(c[0]), "+d"(c[1])                                                                  \
               : "d"(a), "d"(b))
    PLUQ_DMMA(c0); PLUQ_DMMA(c1); PLUQ_DMMA(c2); PLUQ_DMMA(c3);
#undef PLUQ_DMMA
  }
  const double s = c0[0] + c0[1] + c1[0] + c1[1] + c2[0] + c2[1] + c3[0] + c3[1];
  if (s == 12345.678) sink[threadIdx.x] = s;  // keep the work alive
}

// ------------------------------- host side ---------------------------------------------
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

struct TcGemm {
  PFN_encodeTiled encode = nullptr;
  std::string last_error;
  int64_t k_pass_override = 0;  // tests: force multi-pass K splitting
  bool attrs_set[2][3][5][2] = {};
  int epi_warps = 8;            // option tc_epi: epilogue warps of the 1-set (V = 1) kernels (8 or 16)
  int variant = 1;              // TcCfg variant (option tc_cfg)
  int grid_override = 0;        // tests/diagnostics: CTAs of the persistent kernel (option tc_grid)
  int dbg = 0;                  // diagnostics only (option tc_dbg): 1 = skip operand loads after the first ring, 2 = skip the epilogue
  int vec_limbs = 1;            // vectorised limb-split kernels (option tc_vec)
  int pair_split = 1;           // both operands' limb split in one launch (option tc_pair)
  int time_mma = 0;             // option tc_time: time the MMA kernel alone (adds a sync)
  int mn_b = 1;                 // option tc_mnb: MN-major B operand when the tile allows it (no transpose)
  int raster_group = 8;         // option tc_group: tile rows per rasterisation group (0: row-major tiles)
  int c_prefetch = 1;           // option tc_cpf: L2 prefetch of the C tile while its MMAs run
  float mma_ms = 0.f;           // summed MMA-kernel time of the last call when timed
  cudaMemPool_t pool = nullptr; // the owning context's memory pool (limb-plane scratch)
  // option tc_time: MMA-kernel launches, their summed CUDA-event time and algorithmic int8
  // ops (2 m n k L^2 per pass) since the context's last reset_stats (bench roofline)
  int64_t acc_launches = 0;
  double acc_ms = 0.0, acc_ops = 0.0;

  static int limbs(uint32_t p) {
    int bits = 0;
    for (uint32_t v = p - 1; v; v >>= 1) ++bits;
    return bits <= 8 ? 1 : (bits + 7) / 8;
  }
  // largest exact K per pass, multiple of TC_BK: K * L * 255^2 < 2^31
  static int64_t k_pass(int L) {
    int64_t kp = ((int64_t(1) << 31) - 1) / ((int64_t)L * 255 * 255);
    return (kp / TC_BK) * TC_BK;
  }

  int sms = 0;
  int num_sms() {
    if (!sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (sms <= 0) sms = 148;
    }
    return sms;
  }

  void release() {}

  bool load() {
    if (encode) return true;
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      last_error = "cuTensorMapEncodeTiled unavailable";
      return false;
    }
    encode = reinterpret_cast<PFN_encodeTiled>(fn);
    return true;
  }

  bool make_map(CUtensorMap* map, void* base, int64_t inner_bytes, int64_t rows, int box_rows,
                int box_inner = TC_BK) {
    cuuint64_t dims[2] = {(cuuint64_t)inner_bytes, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)inner_bytes};
    cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      last_error = "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")";
      return false;
    }
    return true;
  }

  template <int L, int V, bool MNB, int EPI = 8>
  int launch(const View& c, const View& a, const View& b, const ModP mp, cudaStream_t st, const int* stop,
             int max_ctas) {
    constexpr int BN = TcCfg<L, V>::BN;
    const int m = c.m, n = c.n, k = a.n;
    const int m_pad = (m + TC_BM - 1) / TC_BM * TC_BM;
    const int n_pad = (n + BN - 1) / BN * BN;
    int64_t kp = k_pass_override > 0 ? k_pass_override : k_pass(L);
    kp = (kp / TC_BK) * TC_BK;
    if (kp <= 0) kp = TC_BK;
    const int64_t k_first = std::min<int64_t>(k, kp);
    const int kpad_max = (int)((k_first + TC_BK - 1) / TC_BK * TC_BK);
    uint8_t *da = nullptr, *db = nullptr;
    if (cudaMallocFromPoolAsync((void**)&da, (size_t)L * m_pad * kpad_max, pool, st) != cudaSuccess ||
        cudaMallocFromPoolAsync((void**)&db, (size_t)L * n_pad * kpad_max, pool, st) != cudaSuccess) {
      last_error = "workspace allocation failed";
      return kNoMemory;
    }
    constexpr size_t smem = tc_smem_bytes<L, V, EPI>();
    static_assert(smem <= 232448, "shared memory budget");
    static_assert(V != 2 || (L == 2 && MNB && EPI == 8), "two-pass kernel: two limbs, MN-major B");
    if (!attrs_set[MNB][V][L][EPI == 16]) {
      cudaError_t ae;
      if constexpr (V == 2)
        ae = cudaFuncSetAttribute(tc_modgemm2p_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      else
        ae = cudaFuncSetAttribute(tc_modgemm_kernel<L, V, MNB, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem);
      if (ae != cudaSuccess) {
        last_error = "cannot set shared memory size";
        return kCuda;
      }
      attrs_set[MNB][V][L][EPI == 16] = true;
    }
    for (int64_t k0 = 0; k0 < k; k0 += kp) {
      const int kc = (int)std::min<int64_t>(kp, k - k0);
      const int k_pad = (kc + TC_BK - 1) / TC_BK * TC_BK;
      View as = a.sub(0, (int)k0, m, kc);
      View bs = b.sub((int)k0, 0, kc, n);
      if (vec_limbs && MNB && pair_split) {  // A and B (row-major planes) in one launch
        const int64_t wa = (int64_t)m_pad * (k_pad / 16), wb = (int64_t)k_pad * (n_pad / 16);
        const int gx = (int)std::min<int64_t>((std::max(wa, wb) + 255) / 256, 148 * 16);
        limb_rows16_pair_kernel<<<dim3((unsigned)gx, 2), 256, 0, st>>>(as, da, m_pad, k_pad, bs, db, k_pad, n_pad, L, stop);
      } else {
      if (vec_limbs) {
        const int64_t work = (int64_t)m_pad * (k_pad / 16);
        const int grid = (int)std::min<int64_t>((work + 255) / 256, 148 * 16);
        limb_rows16_kernel<<<grid, 256, 0, st>>>(as, da, L, m_pad, k_pad, stop);
      } else {
        int64_t work = (int64_t)m_pad * (k_pad / 4);
        int grid = (int)std::min<int64_t>((work + 255) / 256, 148 * 32);
        limb_rows_kernel<<<grid, 256, 0, st>>>(as, da, L, m_pad, k_pad, stop);
      }
      if (MNB) {  // B planes row-major (k_pad x n_pad): the same split as A, no transpose
        const int64_t work = (int64_t)k_pad * (n_pad / 16);
        const int grid = (int)std::min<int64_t>((work + 255) / 256, 148 * 16);
        limb_rows16_kernel<<<grid, 256, 0, st>>>(bs, db, L, k_pad, n_pad, stop);
      } else {
        dim3 cgrid(n_pad / 32, k_pad / 32);
        limb_cols_kernel<<<cgrid, 256, 0, st>>>(bs, db, L, n_pad, k_pad, stop);
      }
      }
      CUtensorMap ta, tb;
      const bool okb = MNB ? make_map(&tb, db, n_pad, (int64_t)L * k_pad, TC_BK, BN)
                           : make_map(&tb, db, k_pad, (int64_t)L * n_pad, BN);
      if (!make_map(&ta, da, k_pad, (int64_t)L * m_pad, TC_BM) || !okb) {
        cudaFreeAsync(da, st);
        cudaFreeAsync(db, st);
        return kCuda;
      }
      const int tiles = (n_pad / BN) * (m_pad / TC_BM);
      // max_ctas < 0: one CTA per tile (not persistent), so the grid fills whatever SMs free
      // up while a persistent kernel on another stream holds the rest
      const int grid = max_ctas < 0 ? tiles
                                    : std::min(tiles, max_ctas > 0 ? max_ctas
                                                                   : grid_override > 0 ? grid_override : num_sms());
      cudaEvent_t e0 = nullptr, e1 = nullptr;
      if (time_mma) {
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
      }
      if constexpr (V == 2)
        tc_modgemm2p_kernel<<<grid, TcEpi<8>::THREADS, smem, st>>>(ta, tb, c, m_pad, n_pad, k_pad / TC_BK, mp, stop,
                                                                   dbg, raster_group, c_prefetch);
      else
        tc_modgemm_kernel<L, V, MNB, EPI><<<grid, TcEpi<EPI>::THREADS, smem, st>>>(
            ta, tb, c, m_pad, n_pad, k_pad / TC_BK, mp, stop, dbg, raster_group, c_prefetch);
      if (time_mma) {
        float ms = 0.f;
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        mma_ms += ms;
        acc_ms += ms;
        acc_ops += 2.0 * m * n * (double)kc * L * L;
        ++acc_launches;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
      }
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) {
        last_error = std::string("tc_modgemm launch: ") + cudaGetErrorString(e);
        cudaFreeAsync(da, st);
        cudaFreeAsync(db, st);
        return kCuda;
      }
    }
    cudaFreeAsync(da, st);
    cudaFreeAsync(db, st);
    return kOk;
  }

  int run(const View& c, const View& a, const View& b, const ModP mp, cudaStream_t st, const int* stop = nullptr,
          int max_ctas = 0) {
    mma_ms = 0.f;
    if (c.m == 0 || c.n == 0 || a.n == 0) return kOk;
    if (c.m > (1 << 24) || c.n > (1 << 24)) return kUnsupported;
    if (!load()) return kUnsupported;
    const int L = limbs(mp.p);
    if (variant == 0) {
      switch (L) {
        case 1: return launch<1, 0, false>(c, a, b, mp, st, stop, max_ctas);
        case 2: return launch<2, 0, false>(c, a, b, mp, st, stop, max_ctas);
        case 3: return launch<3, 0, false>(c, a, b, mp, st, stop, max_ctas);
        case 4: return launch<4, 0, false>(c, a, b, mp, st, stop, max_ctas);
      }
    } else {
      switch (L) {
        case 1: return launch<1, 1, false>(c, a, b, mp, st, stop, max_ctas);
        case 2:
          if (mn_b && variant == 2) return launch<2, 2, true>(c, a, b, mp, st, stop, max_ctas);
          if (mn_b && epi_warps == 16) return launch<2, 1, true, 16>(c, a, b, mp, st, stop, max_ctas);
          return mn_b ? launch<2, 1, true>(c, a, b, mp, st, stop, max_ctas)
                      : launch<2, 1, false>(c, a, b, mp, st, stop, max_ctas);
        case 3: return launch<3, 1, false>(c, a, b, mp, st, stop, max_ctas);
        case 4: return launch<4, 1, false>(c, a, b, mp, st, stop, max_ctas);
      }
    }
    return kUnsupported;
  }
};

}  // namespace pluq
