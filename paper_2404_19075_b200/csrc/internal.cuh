// internal.cuh -- context object, kernel parameter blocks and launch helpers shared by the
// libdinr.so translation units (not part of the ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/dinr.h"
#include "philox.cuh"

namespace dinr {

constexpr int kTile = 128;          // samples per tensor-core tile (= TMEM lanes)
constexpr int kChunk = 32;          // samples per ray-sum partial (one warp)
constexpr int kMaxH = 256;

enum TimerClass { T_RAYS = 0, T_FWD = 1, T_LOSS = 2, T_BWD = 3, T_DW = 4, T_ASM = 5, T_PACK = 6, T_AR = 7, T_N = 8 };

// Geometry in the form the kernels use (fp64).
struct GeomParams {
  int beam, n_rows, n_cols, sub_x, sub_z, n_s;
  double sod, odd, dx, dz, cx, cz, r, xs0;
  double zc, zh, tc, th;  // normalization centres / half widths (R11)
  int64_t M;              // number of views
  int jitter;             // N3: sub-pixel jitter on (seed, step below)
  uint32_t seed_lo, seed_hi, step;
  // host-computed reciprocals (correctly rounded, so identical to the device division):
  // inv_sub_* is used only when sub_* is a power of two (then x * (1/sub) == x / sub exactly)
  double ir, izh, inv_sub_x, inv_sub_z, inv_ns;  // inv_ns likewise only for N_s a power of two
};

// Per-ray packed fp32 record (2 x float4), produced by K1, consumed by the MLP kernels:
//   a = (xbar, ybar, zbar, tbar) normalized coordinates of the point at delta_min
//   b = (dxbar, dybar, dzbar, wq) normalized per-sample step and quadrature weight chord/N_s
// Sample j of the ray sits at a.xyz + (j + u_j) b.xyz: u_j = 1/2 (midpoint rule, R8) or the
// N3 stratified jitter (philox.cuh).

// Launch-bound scratch for the tensor-core backward.
struct TcScratch {
  uint16_t *hstash;   // L x n_tiles x (H*128) bf16 images of h_l (layer inputs)
  uint16_t *dstash;   // L x n_tiles x (H*128) bf16 images of delta_l
  uint16_t *zstash;   // (L-1) x n_tiles x (H*128) fp16, chunk-major
  float *head_part;   // grid x (H+1)
  float *dw_part;     // L x nmb x ksplit x 128 x H
  float *db_part;     // L x nmb x ksplit x 128
};

}  // namespace dinr

struct dinr_ctx {
  int device = 0;
  int sm_count = 148;
  std::string err;

  bool have_geom = false;
  dinr_geometry geom{};
  int64_t M = 0;
  int S = 1;
  double *d_views = nullptr;  // M x 3 {cos theta, sin theta, t}
  std::vector<double> h_t;    // view times (host copy, N4)
  // N3 sample placement (dinr_set_sampling)
  int sampling = DINR_MIDPOINT;
  uint64_t seed = 0;
  uint32_t step = 0;

  bool have_field = false;
  dinr_field_desc field{};
  int C = 0, L = 0, H = 0;
  int64_t P = 0;
  float *d_B = nullptr;
  float *d_params = nullptr;
  uint16_t *d_wpack = nullptr;       // bf16 SW128 images of W_l
  uint16_t *d_wpack_half = nullptr;  // same, prescaled by 0.5 (fused kernel)
  size_t wpack_cap = 0, params_cap = 0;

  // scratch (grown on demand)
  void *scratch = nullptr;
  size_t scratch_cap = 0;
  std::vector<size_t> guard_bands;  // DINR_GUARDS: offsets of the 4 KB bands around the plan's buffers
  int *d_flags = nullptr;  // [0] = out-of-range index seen
  float *d_ones = nullptr;
  void *d_prims = nullptr;  // N2 phantom primitives (64 slots)

  // instrumentation
  bool timing = false;
  struct Pending {
    int cls;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> event_pool;
  double acc_ms[dinr::T_N] = {0};
  int64_t acc_n[dinr::T_N] = {0};
  int64_t launches = 0;

  // NCCL
  void *comm = nullptr;
  int rank = 0, world = 1;
};
