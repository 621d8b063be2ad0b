// Shared device helpers for the B200 PLUQ-mod-p path.
//
// Storage: every residue lives in HBM/SMEM as uint32 in [0, p), p < 2^31 prime
// (the reference allows p < 2^26 by default and < 2^31 with
// allow_large_modulus, /root/reference/pkg/src/pluq/field.py:19-21,65-73).
// Products are formed in 64 bits and reduced with a Barrett step.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define PLUQ_HD __host__ __device__ __forceinline__

namespace pluq {

// Status codes crossing the C ABI (mapped to Python exceptions by the wrapper).
enum Status : int {
  kOk = 0,
  kInvalid = 1,       // ValueError
  kZeroDivision = 2,  // ZeroDivisionError
  kCuda = 3,          // RuntimeError (CUDA)
  kNoMemory = 4,      // MemoryError
  kUnsupported = 5,   // NotImplementedError
};

struct ModP {
  uint32_t p;
  uint32_t mu32;     // floor((2^32 - 1) / p) when p < 2^16 (32-bit Barrett), else 0
  uint64_t mu;       // floor((2^64 - 1) / p), Barrett constant
  uint64_t kchunk;   // max number of (p-1)^2 products summable in uint64 without overflow
  const uint32_t* itab32;  // device table of inverses for 2^16 <= p <= 2^25 (a^-1 at index a), or nullptr

  static ModP make(uint32_t p_) {
    ModP m;
    m.p = p_;
    m.mu32 = p_ < 65536u ? 0xffffffffu / p_ : 0u;
    m.mu = ~0ull / p_;
    unsigned __int128 sq = (unsigned __int128)(p_ - 1) * (p_ - 1);
    m.kchunk = sq ? (uint64_t)(((unsigned __int128)~0ull - (unsigned __int128)(p_ - 1)) / sq) : ~0ull;
    if (m.kchunk == 0) m.kchunk = 1;
    m.itab32 = nullptr;
    return m;
  }
};

// x mod p for any 64-bit x.
// Barrett: q = floor(x * mu / 2^64) underestimates floor(x / p) by at most 2, so two
// branch-free conditional subtractions finish the reduction.
PLUQ_HD uint32_t reduce64(uint64_t x, const ModP m) {
#ifdef __CUDA_ARCH__
  uint64_t q = __umul64hi(x, m.mu);
#else
  uint64_t q = (uint64_t)(((unsigned __int128)x * m.mu) >> 64);
#endif
  uint64_t r = x - q * (uint64_t)m.p;
  r = r >= m.p ? r - m.p : r;
  r = r >= m.p ? r - m.p : r;
  return (uint32_t)r;
}

// x mod p for x < 2^32 when p < 2^16: q = floor(x * mu32 / 2^32) is short by at most 2.
PLUQ_HD uint32_t reduce32(uint32_t x, const ModP m) {
#ifdef __CUDA_ARCH__
  uint32_t q = __umulhi(x, m.mu32);
#else
  uint32_t q = (uint32_t)(((uint64_t)x * m.mu32) >> 32);
#endif
  uint32_t r = x - q * m.p;
  r = r >= m.p ? r - m.p : r;
  r = r >= m.p ? r - m.p : r;
  return r;
}

PLUQ_HD uint32_t mulmod(uint32_t a, uint32_t b, const ModP m) {
  if (m.mu32) return reduce32(a * b, m);  // a, b < p < 2^16: the product fits 32 bits
  return reduce64((uint64_t)a * b, m);
}

PLUQ_HD uint32_t addmod(uint32_t a, uint32_t b, const ModP m) {
  uint32_t s = a + b;  // a, b < 2^31 so no wrap
  return s >= m.p ? s - m.p : s;
}

PLUQ_HD uint32_t submod(uint32_t a, uint32_t b, const ModP m) {
  return a >= b ? a - b : a + (m.p - b);
}

// Multiplicative inverse via extended Euclid (field.py:41-52); a != 0 mod p.
// 32-bit arithmetic throughout: remainders are < p < 2^31 and |Bezout coefficients| <= p.
PLUQ_HD uint32_t invmod(uint32_t a, const ModP m) {
#ifdef __CUDA_ARCH__
  // primes of 17..25 bits (cfg4: 23 bits): one table load (L2-resident) instead of ~40 dependent
  // divisions on the pivot chain of every base-case / diagonal-block / TRSM kernel
  if (m.itab32) return __ldg(m.itab32 + a);
#endif
  uint32_t old_r = a, r = m.p;
  int32_t old_s = 1, s = 0;
  while (r) {
    uint32_t q = old_r / r;
    uint32_t t = old_r - q * r; old_r = r; r = t;
    int32_t ts = old_s - (int32_t)q * s; old_s = s; s = ts;
  }
  return old_s < 0 ? (uint32_t)(old_s + (int32_t)m.p) : (uint32_t)old_s;
}

// Row-major view into a larger row-major matrix (global or shared; generic pointer).
struct View {
  uint32_t* a;
  int64_t ld;
  int m, n;
  PLUQ_HD uint32_t* row(int i) const { return a + (int64_t)i * ld; }
  PLUQ_HD uint32_t& at(int i, int j) const { return a[(int64_t)i * ld + j]; }
  PLUQ_HD View sub(int r0, int c0, int mm, int nn) const {
    View v{a + (int64_t)r0 * ld + c0, ld, mm, nn};
    return v;
  }
};

// Closed-form OpCounts charges of the reference kernels (kernels.py:1-16, 38-120).
struct Counts {
  unsigned long long mul, add, inv, red;
};

PLUQ_HD void charge_mm(Counts& c, long long m, long long n, long long k) {
  if (k == 0 || m == 0 || n == 0) return;
  c.red += m * n; c.mul += m * n * k; c.add += m * n * k;
}
PLUQ_HD void charge_trsm_l(Counts& c, long long r, long long n) {
  if (r == 0 || n == 0) return;
  c.red += r * n; c.mul += n * (r * (r - 1) / 2); c.add += n * (r * (r - 1) / 2);
}
PLUQ_HD void charge_trsm_u(Counts& c, long long m, long long r) {
  if (r == 0) return;
  c.inv += r;
  if (m == 0) return;
  c.red += 2 * m * r; c.mul += m * (r * (r + 1) / 2); c.add += m * (r * (r - 1) / 2);
}

}  // namespace pluq
