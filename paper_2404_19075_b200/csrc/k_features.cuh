// k_features.cuh -- GRFF input encoding of one sample (a5/a6 of the hot path), shared by the
// fused training kernels and the dW GEMM (which recomputes layer 0's input instead of
// re-reading it from HBM).  gamma(x) = [cos(2 pi B x), sin(2 pi B x)] (eq:grff)
// evaluated at the ray-sample coordinates from the fp32 ray records (R6, R9).
#pragma once
#include "internal.cuh"
#include "k_geometry.cuh"
#include "ptx_sm100.cuh"

namespace dinr {

// (t, z, y, x) coordinates of global sample g = ray * n_s + j, sample j of the ray in its stratum
// (rec32[2 ray] = origin + t, rec32[2 ray + 1] = step + quadrature weight).  Zero if !valid.
__device__ __forceinline__ float4 grff_coords(const float4 *__restrict__ rec32, int64_t g, int lg_ns, int n_s,
                                              bool valid, const Jitter &jt) {
  float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
  if (valid) {
    // N_s a power of two: shifts; otherwise (split path, e.g. N_s = 96) a division
    const int64_t ray = (n_s & (n_s - 1)) == 0 ? g >> lg_ns
                        : ((g >> 32) == 0 ? (int64_t)((uint32_t)g / (uint32_t)n_s) : g / n_s);
    const uint32_t j = (uint32_t)(g - ray * n_s);
    const float jj = (float)j + sample_offset(jt, ray, j);  // midpoint (R8) or N3 jitter
    const float4 ra = rec32[2 * ray], rv = rec32[2 * ray + 1];
    r.x = ra.w;
    r.y = ra.z + jj * rv.z;
    r.z = ra.y + jj * rv.y;
    r.w = ra.x + jj * rv.x;
  }
  return r;
}

// The same coordinates split into a load (issued early, e.g. one tile ahead) and the arithmetic.
struct RayRec {
  float4 a, b;
};
__device__ __forceinline__ RayRec grff_fetch(const float4 *__restrict__ rec32, int64_t g, int lg_ns, bool valid) {
  RayRec r;
  if (valid) {
    const int64_t ray = g >> lg_ns;
    r.a = rec32[2 * ray];
    r.b = rec32[2 * ray + 1];
  } else {
    r.a = r.b = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  return r;
}
__device__ __forceinline__ float4 grff_coords_from(const RayRec &rr, int64_t g, int lg_ns, int n_s, bool valid,
                                                   const Jitter &jt) {
  float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
  if (valid) {
    const int64_t ray = g >> lg_ns;
    const uint32_t j = (uint32_t)(g & (n_s - 1));
    const float jj = (float)j + sample_offset(jt, ray, j);
    r.x = rr.a.w;
    r.y = rr.a.z + jj * rr.b.z;
    r.z = rr.a.y + jj * rr.b.y;
    r.w = rr.a.x + jj * rr.b.x;
  }
  return r;
}

// Frequencies c0 .. c0+7 (B rows as float4 in shared memory): packed bf16 cos / sin pairs.
__device__ __forceinline__ void grff8(const float4 *sB4, int c0, float4 rb, uint32_t (&pc)[4], uint32_t (&ps)[4]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    float cs[2], sn[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const float4 bb = sB4[c0 + 2 * q + e];
      const float phi = bb.x * rb.x + bb.y * rb.y + bb.z * rb.z + bb.w * rb.w;
      const float fr = phi - rintf(phi);  // phase mod 1: keeps __sincosf in its accurate range
      __sincosf(6.283185307179586f * fr, &sn[e], &cs[e]);
    }
    pc[q] = pack_bf16x2(cs[0], cs[1]);
    ps[q] = pack_bf16x2(sn[0], sn[1]);
  }
}

// N4 voxel grid slab: voxel v of the launch -> (i, j, k) = (v % nx, (v / nx) % ny, k0 + v / (nx ny)),
// centre (x0 + (i + 1/2) vx, y0 + (j + 1/2) vy, z0 + (k + 1/2) vz) at normalized time tbar.
struct VoxGrid {
  int64_t nx, ny, k0;
  double x0, y0, z0, vx, vy, vz;
  double xs0, r, zc, zh;  // normalization (R11) and FOV cylinder
  float tbar;
};

// Normalized (t, z, y, x) of voxel v (fp64 centre, rounded once to fp32) and whether the centre
// lies in the FOV cylinder (x - x_s0)^2 + y^2 <= r^2, decided in fp64 without contraction.
__device__ __forceinline__ float4 voxel_coords(const VoxGrid &vg, int64_t v, bool &inside) {
  int64_t i, j, k;
  if ((v >> 32) == 0 && (vg.nx >> 16) == 0 && (vg.ny >> 16) == 0) {  // 32-bit divisions (the 64-bit ones are calls)
    const uint32_t v32 = (uint32_t)v, nx = (uint32_t)vg.nx, ny = (uint32_t)vg.ny;
    const uint32_t r = v32 / nx;
    i = v32 - r * nx;
    j = r % ny;
    k = vg.k0 + r / ny;
  } else {
    i = v % vg.nx;
    j = (v / vg.nx) % vg.ny;
    k = vg.k0 + v / (vg.nx * vg.ny);
  }
  const double x = dadd(vg.x0, dmul(dadd((double)i, 0.5), vg.vx));
  const double y = dadd(vg.y0, dmul(dadd((double)j, 0.5), vg.vy));
  const double z = dadd(vg.z0, dmul(dadd((double)k, 0.5), vg.vz));
  const double px = dsub(x, vg.xs0);
  inside = dadd(dmul(px, px), dmul(y, y)) <= dmul(vg.r, vg.r);
  float4 r;
  r.x = vg.tbar;
  r.y = vg.zh > 0.0 ? (float)__ddiv_rn(dsub(z, vg.zc), vg.zh) : 0.f;
  r.z = (float)__ddiv_rn(y, vg.r);
  r.w = (float)__ddiv_rn(px, vg.r);
  return r;
}

}  // namespace dinr
