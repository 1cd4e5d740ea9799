// k_phantom.cuh -- NEXT row N2: analytic-phantom projector with transmission-space noise.
//
// Exact line integrals (no quadrature) of ellipsoidal primitives along every sub-ray of a
// pixel, on the K1 fp64 ray records (ray_fp64), then the BEER / LINEAR combine in fp64:
//   indicator  mu inside ellipsoid:   value * s * |chord-in-ellipsoid|           (eq:parlineint)
//   smooth     mu_c (1 - rho^2)^2:    s mu_c A^2 [h^4 u - 2/3 h^2 u^3 + u^5/5]
//   Gaussian   A exp(-rho^2/2):       s A e^{-rmin2/2} sqrt(pi/(2A)) [erf-difference]
// with rho^2(delta) = A delta^2 + B delta + C in the ray parameter, truncated to
// [delta_min, delta_max] (the FOV chord).  Primitives move linearly in time (c0 + v t,
// a0 + adot t), evaluated at the view time t_k (the object is static during one exposure,
// P:153-154).  Optional noise (eq:forwmod P:261-272 with the Results' transmission-space
// convention, R24): T = e^{-f}, T' = max(T + frac sqrt(T) g, 1e-8), y = -ln T', g ~ N(0,1)
// from a counter-based generator keyed by (seed, pixel index).
#pragma once
#include "internal.cuh"
#include "k_geometry.cuh"

namespace dinr {

struct PrimDev {
  int kind;
  double value;
  double c0[3], vel[3], a0[3], arate[3];
};

__device__ double phantom_line_integral(const PrimDev *__restrict__ prims, int np, const double *o, const double *d,
                                        double dmin, double dmax, double t) {
  if (!(dmax > dmin)) return 0.0;
  const double s = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
  double total = 0.0;
  for (int q = 0; q < np; ++q) {
    const PrimDev &pr = prims[q];
    double A = 0.0, Bq = 0.0, Cq = 0.0;
    for (int k = 0; k < 3; ++k) {
      const double ck = pr.c0[k] + pr.vel[k] * t, ak = pr.a0[k] + pr.arate[k] * t;
      const double dk = d[k] / ak, ok = (o[k] - ck) / ak;
      A += dk * dk;
      Bq += 2.0 * ok * dk;
      Cq += ok * ok;
    }
    const double dc = -Bq / (2.0 * A);
    const double rmin2 = Cq - Bq * Bq / (4.0 * A);
    if (pr.kind == 2) {
      const double k2 = sqrt(0.5 * A);
      const double x1 = k2 * (dmin - dc), x2 = k2 * (dmax - dc);
      double diff;
      if (x1 >= 0.0)
        diff = erfc(x1) - erfc(x2);
      else if (x2 <= 0.0)
        diff = erfc(-x2) - erfc(-x1);
      else
        diff = erf(x2) - erf(x1);
      total += s * pr.value * exp(-0.5 * rmin2) * sqrt(3.141592653589793 / (2.0 * A)) * diff;
      continue;
    }
    if (rmin2 >= 1.0) continue;
    const double h = sqrt((1.0 - rmin2) / A);
    const double lo = fmax(dc - h, dmin) - dc, hi = fmin(dc + h, dmax) - dc;
    if (!(hi > lo)) continue;
    if (pr.kind == 0) {
      total += s * pr.value * (hi - lo);
    } else {
      const double h2 = h * h;
      auto F = [&](double u) { return h2 * h2 * u - (2.0 / 3.0) * h2 * u * u * u + u * u * u * u * u / 5.0; };
      total += s * pr.value * A * A * (F(hi) - F(lo));
    }
  }
  return total;
}

// splitmix64-based counter generator -> one standard normal (Box-Muller)
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ double normal_from_counter(uint64_t seed, uint64_t ctr) {
  const uint64_t a = splitmix64(seed ^ splitmix64(2 * ctr)), b = splitmix64(seed ^ splitmix64(2 * ctr + 1));
  const double u1 = ((double)(a >> 11) + 0.5) * (1.0 / 9007199254740992.0);
  const double u2 = (double)(b >> 11) * (1.0 / 9007199254740992.0);
  return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}

__global__ void k_phantom_project(GeomParams gp, const double *__restrict__ views, const int64_t *__restrict__ idx,
                                  int64_t n, const PrimDev *__restrict__ prims, int np, int combine,
                                  double noise_frac, uint64_t seed, float *__restrict__ fhat,
                                  float *__restrict__ p_sub, int *__restrict__ flags) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int S = gp.sub_x * gp.sub_z;
  double pv[kMaxS];
  bool ok = true;
  for (int s = 0; s < S; ++s) {
    double r[9], tk = 0.0;
    if (!ray_fp64(gp, views, idx[p], s, r, tk)) {
      ok = false;
      pv[s] = 0.0;
      continue;
    }
    pv[s] = r[8] > 0.0 ? phantom_line_integral(prims, np, r, r + 3, r[6], r[7], tk) : 0.0;
    if (p_sub) p_sub[p * S + s] = (float)pv[s];
  }
  if (!ok) {
    atomicOr(flags, 1);
    for (int s = 0; s < S; ++s) pv[s] = 0.0;
  }
  double f;
  if (combine == DINR_LINEAR) {
    double a = 0.0;
    for (int s = 0; s < S; ++s) a += pv[s];
    f = a / (double)S;
  } else {
    double m = pv[0];
    for (int s = 1; s < S; ++s) m = fmin(m, pv[s]);
    double T = 0.0;
    for (int s = 0; s < S; ++s) T += exp(-(pv[s] - m));
    f = m - log(T / (double)S);
  }
  if (noise_frac > 0.0) {
    const double T = exp(-f);
    const double Tn = fmax(T + noise_frac * sqrt(T) * normal_from_counter(seed, (uint64_t)idx[p]), 1e-8);
    f = -log(Tn);
  }
  fhat[p] = (float)f;
}

}  // namespace dinr
