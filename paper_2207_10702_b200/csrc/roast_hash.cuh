// roast_hash.cuh — library hash family (implementation #2), __host__ __device__.
//
// Written from the mapping definition in include/roast.h (PAPER.md P:268-289,
// P:315; readings R1-R3, R8 of DESIGN.md).  Shares no code with oracle/.
// Device path: 128-bit product via __umul64hi, Mersenne fold, no division
// except the final `mod R`.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define RH_HD __host__ __device__ __forceinline__
#else
#define RH_HD inline
#endif

namespace roast {

constexpr uint64_t kP61 = (uint64_t(1) << 61) - 1;

RH_HD uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// a * b mod (2^61 - 1) for a, b < 2^61.
RH_HD uint64_t mulmod61(uint64_t a, uint64_t b) {
  uint64_t lo, hi;
#ifdef __CUDA_ARCH__
  lo = a * b;
  hi = __umul64hi(a, b);
#else
  unsigned __int128 p = (unsigned __int128)a * b;
  lo = (uint64_t)p;
  hi = (uint64_t)(p >> 64);
#endif
  // p = hi * 2^64 + lo;  p mod P = (p & P) + (p >> 61)  (one fold, then one subtract)
  uint64_t s = (lo & kP61) + ((hi << 3) | (lo >> 61));
  return s >= kP61 ? s - kP61 : s;
}

RH_HD uint64_t addmod61(uint64_t a, uint64_t b) {
  uint64_t s = a + b;
  return s >= kP61 ? s - kP61 : s;
}

struct PolyCoef {
  uint64_t c[4];  // c0..c3, each < P
};

RH_HD PolyCoef make_coef(uint64_t seed, uint32_t module, uint32_t role) {
  PolyCoef p;
  for (uint32_t r = 0; r < 4; ++r) {
    uint64_t tag = (uint64_t(module) << 8) | (uint64_t(role) << 4) | r;
    p.c[r] = mix64(seed ^ mix64(tag)) % kP61;
  }
  return p;
}

// Horner: ((c3 k + c2) k + c1) k + c0 mod P, key < 2^60.
RH_HD uint64_t poly61(const PolyCoef& p, uint64_t key) {
  uint64_t v = p.c[3];
  v = addmod61(mulmod61(v, key), p.c[2]);
  v = addmod61(mulmod61(v, key), p.c[1]);
  v = addmod61(mulmod61(v, key), p.c[0]);
  return v;
}

RH_HD uint64_t tile_key(uint32_t x, uint32_t y) { return (uint64_t(x) << 32) | y; }

// Exact v mod R for v < 2^61 by an invariant-divisor reciprocal (Granlund & Montgomery
// 1994, Thm 4.2 with N = 61): l = ceil(log2 R), m = ceil(2^(61+l) / R) < 2^63,
// q = floor(v m / 2^(61+l)) = floor(v / R) for every v < 2^61.  The device path avoids
// the ~100-instruction software 64-bit division of `%`.
struct ModReciprocal {
  uint64_t R = 1, m = 0;
  uint32_t s = 0;  // 61 + l
  void init(uint64_t r) {
    R = r;
    uint32_t l = 0;
    while ((uint64_t(1) << l) < r) ++l;
    s = 61 + l;
    // m = ceil(2^s / R) with 128-bit arithmetic (host only)
    unsigned __int128 p = (unsigned __int128)1 << s;
    m = uint64_t((p + R - 1) / R);
  }
};

RH_HD uint64_t mod_recip(uint64_t v, const ModReciprocal& d) {
  uint64_t lo, hi;
#ifdef __CUDA_ARCH__
  lo = v * d.m;
  hi = __umul64hi(v, d.m);
#else
  unsigned __int128 p = (unsigned __int128)v * d.m;
  lo = (uint64_t)p;
  hi = (uint64_t)(p >> 64);
#endif
  const uint64_t q = d.s >= 64 ? (hi >> (d.s - 64)) : ((hi << (64 - d.s)) | (lo >> d.s));
  return v - q * d.R;
}

struct ModuleHash {
  PolyCoef off, sgn;
  uint64_t R;       // number of legal aligned positions
  uint32_t align;   // A
  uint32_t use_sign;
  ModReciprocal rdiv;  // v mod R without division (set by set_range)
  uint64_t base = 0;   // first element of the module's memory: 0 under GMS, its segment under LMS

  void set_range(uint64_t r) {
    R = r;
    rdiv.init(r);
  }
  RH_HD uint64_t offset(uint64_t key) const { return base + uint64_t(align) * mod_recip(poly61(off, key), rdiv); }
  RH_HD int sign(uint64_t key) const {
    return (use_sign && (poly61(sgn, key) & 1)) ? -1 : 1;
  }
};

}  // namespace roast
