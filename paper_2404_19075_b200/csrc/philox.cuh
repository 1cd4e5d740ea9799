// philox.cuh -- N3 counter-based generator: Philox4x32-10 (Salmon, Moraes, Dror,
// Shaw, SC'11) and the stratified-jitter offsets derived from it.  The oracle implements the same
// generator independently (the fp64 oracle, test infrastructure); both sides draw
//   sample j of global ray R:  u = u01(philox((j, R lo, R hi, step), (seed lo, seed hi)).x)
//   sub-pixel offset of R:     (ux, uz) = u01 of .x, .y for counter word 0 = 0xFFFFFFFF
// with u01(x) = (x >> 8) 2^-24 (exact in fp32 and fp64).  R = pixel index * S + s.
#pragma once
#include <cstdint>

namespace dinr {

__host__ __device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c.x, p1 = (uint64_t)0xCD9E8D57u * c.z;
    c = make_uint4((uint32_t)(p1 >> 32) ^ c.y ^ k.x, (uint32_t)p1, (uint32_t)(p0 >> 32) ^ c.w ^ k.y, (uint32_t)p0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

__host__ __device__ __forceinline__ float u01f(uint32_t x) { return (float)(x >> 8) * 5.9604644775390625e-08f; }

// Sampling state handed to every kernel that places samples (off: rid == nullptr, midpoint rule).
struct Jitter {
  const uint2 *rid;  // global ray id (lo, hi) of each batch ray, written by K1
  uint32_t seed_lo, seed_hi, step;
};

// Offset of sample j inside its stratum of batch ray `ray` (1/2 = midpoint rule, R8).
__device__ __forceinline__ float sample_offset(const Jitter &jt, int64_t ray, uint32_t j) {
  if (jt.rid == nullptr) return 0.5f;
  const uint2 id = jt.rid[ray];
  return u01f(philox4x32_10(make_uint4(j, id.x, id.y, jt.step), make_uint2(jt.seed_lo, jt.seed_hi)).x);
}

}  // namespace dinr
