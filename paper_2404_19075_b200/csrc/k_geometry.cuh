// k_geometry.cuh -- K1 ray setup (north_star subsystem (1)).
//
// One thread per sub-ray.  fp64 with explicitly rounded intrinsics (__dadd_rn, __dmul_rn,
// __ddiv_rn, __dsqrt_rn) so no FMA contraction occurs and the operation order is the
// one written in DESIGN.md "Ray geometry" (the oracle writes the same formulas in plain C
// compiled with -ffp-contract=off; cos/sin come from the host libm via the view table):
//   a1 decode    i = m N + n, row = n / n_cols, col = n % n_cols        (R13)
//   a3 endpoints x_d = -C_x + (col + (u+ux)/D_x) dx, y_d = odd,
//                z_d = -C_z + (row + (v+uz)/D_z) dz
//                ux = uz = 1/2 (midpoint, R8) or the N3 Philox jitter (philox.cuh)
//                source cone (0,-sod,0) / fan (0,-sod,z_d) / parallel (x_d,-sod,z_d)
//                                                                        (R9, R10)
//   a4 bounds    a = ex^2+ey^2, b = 2(px ex + y_s ey), c = (px^2 + y_s^2) - r^2,
//                disc = b^2 - 4ac, roots (-b -+ sqrt(disc))/(2a) clamped to [0,1]
//                                                                        (R21)
//                arc length s = sqrt(a + ez^2) (P:155-172 read as Euclidean, R1),
//                chord = s (delta_max - delta_min)
//   a2 rotation  x' = (x c - y s) + (x_s0 - x_s0 c), y' = (x s + y c) - x_s0 s
#pragma once
#include "internal.cuh"

namespace dinr {

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

__device__ __forceinline__ void rot_cs(double x, double y, double c, double s, double xs0, double &xo,
                                       double &yo) {
  xo = dadd(dsub(dmul(x, c), dmul(y, s)), dsub(xs0, dmul(xs0, c)));
  yo = dsub(dadd(dmul(x, s), dmul(y, c)), dmul(xs0, s));
}

// One sub-ray's fp64 record {o, d, delta_min, delta_max, chord}; returns false for an
// out-of-range pixel index.  Shared by K1 and the analytic phantom projector (N2).
__device__ __forceinline__ bool ray_fp64(const GeomParams &gp, const double *__restrict__ views, int64_t i, int s,
                                         double r[9], double &tk) {
  int u = s % gp.sub_x, v = s / gp.sub_x;
  int64_t N = (int64_t)gp.n_rows * gp.n_cols;
  if (i < 0 || i >= gp.M * N) return false;
  int64_t k, row, col;
  if ((i >> 32) == 0 && (N >> 32) == 0) {  // 32-bit divisions (the 64-bit ones are subroutine calls)
    const uint32_t i32 = (uint32_t)i, N32 = (uint32_t)N, nc = (uint32_t)gp.n_cols;
    const uint32_t k32 = i32 / N32, nn = i32 - k32 * N32, r32 = nn / nc;
    k = k32;
    row = r32;
    col = nn - r32 * nc;
  } else {
    const int64_t nn = i % N;
    k = i / N;
    row = nn / gp.n_cols;
    col = nn % gp.n_cols;
  }
  double ck = views[3 * k], sk = views[3 * k + 1];
  tk = views[3 * k + 2];

  // sub-pixel offset in its cell: centre (R8) or the N3 jitter of global ray R = i S + s
  double ux = 0.5, uz = 0.5;
  if (gp.jitter) {
    const uint64_t R = (uint64_t)i * (uint64_t)(gp.sub_x * gp.sub_z) + (uint64_t)s;
    const uint4 o = philox4x32_10(make_uint4(0xFFFFFFFFu, (uint32_t)R, (uint32_t)(R >> 32), gp.step),
                                  make_uint2(gp.seed_lo, gp.seed_hi));
    ux = (double)u01f(o.x);
    uz = (double)u01f(o.y);
  }
  // (u + ux) / D_x: a multiply by the exact reciprocal when D_x is a power of two (same result)
  const double fx = (gp.sub_x & (gp.sub_x - 1)) == 0 ? dmul(dadd((double)u, ux), gp.inv_sub_x)
                                                     : __ddiv_rn(dadd((double)u, ux), (double)gp.sub_x);
  const double fz = (gp.sub_z & (gp.sub_z - 1)) == 0 ? dmul(dadd((double)v, uz), gp.inv_sub_z)
                                                     : __ddiv_rn(dadd((double)v, uz), (double)gp.sub_z);
  double xd = dadd(-gp.cx, dmul(dadd((double)col, fx), gp.dx));
  double yd = gp.odd;
  double zd = dadd(-gp.cz, dmul(dadd((double)row, fz), gp.dz));
  double xs, ys = -gp.sod, zs;
  if (gp.beam == DINR_CONE) {
    xs = 0.0;
    zs = 0.0;
  } else if (gp.beam == DINR_FAN) {
    xs = 0.0;
    zs = zd;
  } else {
    xs = xd;
    zs = zd;
  }
  double ex = dsub(xd, xs), ey = dsub(yd, ys), px = dsub(xs, gp.xs0);
  double a = dadd(dmul(ex, ex), dmul(ey, ey));
  double b = dmul(2.0, dadd(dmul(px, ex), dmul(ys, ey)));
  double c = dsub(dadd(dmul(px, px), dmul(ys, ys)), dmul(gp.r, gp.r));
  double disc = dsub(dmul(b, b), dmul(dmul(4.0, a), c));
  double dmin = 0.0, dmax = 0.0;
  if (!(disc < 0.0)) {
    double q = __dsqrt_rn(disc);
    double lo = __ddiv_rn(dsub(-b, q), dmul(2.0, a));
    double hi = __ddiv_rn(dadd(-b, q), dmul(2.0, a));
    dmin = fmin(fmax(lo, 0.0), 1.0);
    dmax = fmin(fmax(hi, 0.0), 1.0);
  }
  double ez = dsub(zd, zs);
  double sarc = __dsqrt_rn(dadd(a, dmul(ez, ez)));
  double chord = dmul(sarc, dsub(dmax, dmin));
  double xsk, ysk, xdk, ydk;
  rot_cs(xs, ys, ck, sk, gp.xs0, xsk, ysk);
  rot_cs(xd, yd, ck, sk, gp.xs0, xdk, ydk);
  r[0] = xsk;
  r[1] = ysk;
  r[2] = zs;
  r[3] = dsub(xdk, xsk);
  r[4] = dsub(ydk, ysk);
  r[5] = ez;
  r[6] = dmin;
  r[7] = dmax;
  r[8] = chord;
  return true;
}

__global__ void k_ray_setup(GeomParams gp, const double *__restrict__ views, const int64_t *__restrict__ idx,
                            int64_t n, double *__restrict__ rec64, float4 *__restrict__ rec32,
                            uint2 *__restrict__ rid, int *__restrict__ flags, float *__restrict__ wq) {
  const int S = gp.sub_x * gp.sub_z;
  int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= n * S) return;
  const int64_t p = (gid >> 32) == 0 ? (int64_t)((uint32_t)gid / (uint32_t)S) : gid / S;
  int s = (int)(gid - p * S);
  double rr[9], tk;
  if (rid) {  // global ray id, keys the N3 sample offsets in the MLP kernels
    const uint64_t R = (uint64_t)idx[p] * (uint64_t)S + (uint64_t)s;
    rid[gid] = make_uint2((uint32_t)R, (uint32_t)(R >> 32));
  }
  if (!ray_fp64(gp, views, idx[p], s, rr, tk)) {
    atomicOr(flags, 1);
    if (rec64)
      for (int q = 0; q < 9; ++q) rec64[gid * 9 + q] = 0.0;
    if (rec32) {
      rec32[2 * gid] = make_float4(0.f, 0.f, 0.f, 0.f);
      rec32[2 * gid + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (wq) wq[gid] = 0.f;
    return;
  }
  const double ox = rr[0], oy = rr[1], oz = rr[2], dx = rr[3], dy = rr[4], dz = rr[5];
  const double dmin = rr[6], dmax = rr[7], chord = rr[8];
  if (rec64)
    for (int q = 0; q < 9; ++q) rec64[gid * 9 + q] = rr[q];
  if (rec32) {
    // Normalized entry point and per-sample step (R11); weight chord/N_s (R7).
    const double ir = gp.ir, izh = gp.izh;  // host-computed 1/r, 1/z_h (same rounding as here)
    double ex0 = ox + dmin * dx, ey0 = oy + dmin * dy, ez0 = oz + dmin * dz;
    const bool ns_pow2 = (gp.n_s & (gp.n_s - 1)) == 0;  // then x / N_s == x * (1 / N_s) exactly
    double step = ns_pow2 ? (dmax - dmin) * gp.inv_ns : (dmax - dmin) / (double)gp.n_s;
    float tb = gp.th > 0.0 ? (float)((tk - gp.tc) / gp.th) : 0.f;
    bool hit = chord > 0.0;
    rec32[2 * gid] = make_float4((float)((ex0 - gp.xs0) * ir), (float)(ey0 * ir), (float)((ez0 - gp.zc) * izh), tb);
    const float w = hit ? (float)(ns_pow2 ? chord * gp.inv_ns : chord / (double)gp.n_s) : 0.f;
    rec32[2 * gid + 1] = make_float4((float)(step * dx * ir), (float)(step * dy * ir), (float)(step * dz * izh), w);
    if (wq) wq[gid] = w;  // compact copy for the pixel combine (one 4-byte read per ray)
  }
}

}  // namespace dinr
