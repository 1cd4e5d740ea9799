// k_sampler.cuh -- N1 batch sampler ("we randomly choose a subset
// Omega_k of projection indices", epochs P:3333-3336; without replacement through a per-epoch
// permutation, SPEC S:389 / S:412; reading R27 in DESIGN.md).
//
// Epoch e visits the D positions of a process's shard in the order perm_e(0), perm_e(1), ...,
// where perm_e is a bijection of [0, D): an 8-round balanced Feistel network on 2h bits
// (h >= 1 the smallest with 4^h >= D) whose round function is Philox4x32-10 --
//   x = (lh << h) | rh;  round r: (lh, rh) <- (rh, lh ^ (philox((rh, r, e lo, e hi),
//                                                       (seed lo, seed hi ^ 0x9E3779B9)).x & mask))
// -- applied again while the value is >= D (cycle walking: a bijection of [0, 4^h) restricted to
// the orbit walk stays a bijection of [0, D)).  One thread per batch pixel; the pixel's measured
// value is gathered from the caller's y source in the same pass.
#pragma once
#include <cstdint>

#include "philox.cuh"

namespace dinr {

struct SampleArgs {
  int64_t N;             // pixels per view
  int64_t D;             // shard size (positions)
  int64_t base;          // position of batch pixel 0 in the epoch's visiting order (before mod D)
  int64_t n;             // pixels in the batch
  int h;                 // Feistel half width (bits)
  int mode;              // 0: view shard (rank, rank + world, ...), 1: global permutation
  int rank, world;
  uint2 key;             // (seed lo, seed hi ^ 0x9E3779B9)
  uint32_t e_lo, e_hi;   // epoch
  const float *y_src;    // view shard (mode 0, view by view) or all M N pixels (mode 1); may be null
  int64_t *idx;          // out: pixel indices i = k N + n
  float *y;              // out: y_src at the sampled pixels (when y_src != null)
};

__device__ __forceinline__ uint64_t feistel8(uint64_t x, const SampleArgs &a) {
  const uint64_t mask = (1ull << a.h) - 1ull;
  uint64_t lh = x >> a.h, rh = x & mask;
#pragma unroll
  for (uint32_t r = 0; r < 8; ++r) {
    const uint4 o = philox4x32_10(make_uint4((uint32_t)rh, r, a.e_lo, a.e_hi), a.key);
    const uint64_t nr = lh ^ ((uint64_t)o.x & mask);
    lh = rh;
    rh = nr;
  }
  return (lh << a.h) | rh;
}

__global__ void k_sample_batch(SampleArgs a) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.n) return;
  uint64_t x = (uint64_t)((a.base + j) % a.D);
  do {
    x = feistel8(x, a);
  } while (x >= (uint64_t)a.D);
  const int64_t q = (int64_t)x;
  int64_t i;
  if (a.mode == 0) {
    const int64_t view = a.rank + (int64_t)a.world * (q / a.N);
    i = view * a.N + q % a.N;
  } else {
    i = q;
  }
  a.idx[j] = i;
  if (a.y_src) a.y[j] = a.y_src[q];
}

}  // namespace dinr
