/*
 * dinr_oracle.h -- fp64 CPU ORACLE for the DINR differentiable forward projector.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load liboracle.so.  The product path
 * (paper_2404_19075_b200/, libdinr.so) never includes, links or calls anything here,
 * and this file shares no code, header, constant or helper with it.
 *
 * Citations: "P:n" = line n of /root/reference/PAPER.md (the paper text),
 * "S:n" = line n of SPEC.md, "R#" = reading # of DESIGN.md section "Readings".
 *
 * Every function follows the paper's algorithm step by step, in fp64, in plain loops
 * (compiled -O2 -ffp-contract=off so no FMA contraction changes the rounding).
 */
#ifndef DINR_ORACLE_H
#define DINR_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Scanner geometry, P:53-106 (C_ij, rotation), P:2842-2862 (cone placement),
 * plus the normalization box of P:440-445 (R11: explicit inputs). */
typedef struct {
  int32_t beam;      /* 0 parallel, 1 fan, 2 cone                              */
  int32_t n_rows;    /* detector rows (index j of C_ij, z)                      */
  int32_t n_cols;    /* detector cols (index i of C_ij, x)                      */
  int32_t sub_x;     /* D_x sub-pixels along x                      */
  int32_t sub_z;     /* D_z sub-pixels along z                                  */
  int32_t n_s;       /* samples per ray N_s (R8: fixed count, midpoint rule)     */
  double sod, odd;   /* |y_s|, |y_d|                                */
  double dx, dz;     /* Delta_x, Delta_z                                        */
  double cx, cz;     /* C_x, C_z                                                */
  double r;          /* FOV cylinder radius                       */
  double xs0;        /* rotation centre x_s0                          */
  double z_lo, z_hi; /* z normalization range (R11)                              */
  double t_lo, t_hi; /* t normalization range (R11)                              */
  /* N3 ("randomly sampled coordinates"): 0 = midpoint rule (R8),
   * 1 = stratified jitter of the sub-pixel position and of each sample in its stratum,
   * uniforms from Philox4x32-10 keyed by seed, counter (j | 0xFFFFFFFF, ray lo, ray hi, step). */
  int32_t sampling;
  uint32_t step;
  uint64_t seed;
} or_geom;

/* Field (DINR network) description. */
typedef struct {
  int32_t C;         /* GRFF frequencies; width H = 2C                           */
  int32_t L;         /* hidden FC+Swish layers                                   */
  int32_t combine;   /* 0 = BEER (eq:beerstransavg), 1 = LINEAR (eq:beersattenavg) */
  int32_t pad;
  double mu0;        /* LAC scale (eq:weightfactors); applied once (R6) */
} or_field;

/* Analytic phantom primitive (oracle pins, O14).  Axis-aligned in the object frame;
 * centre and semi-axes move linearly in time: c(t) = c0 + vel*t, a(t) = a0 + arate*t. */
typedef struct {
  int32_t kind;      /* 0 indicator ellipsoid, 1 smooth (1-rho^2)^2 ellipsoid, 2 Gaussian */
  int32_t pad;
  double value;      /* mu (indicator), mu_c (smooth), amplitude A (Gaussian)     */
  double c0[3];      /* centre (x,y,z) at t=0                                     */
  double vel[3];
  double a0[3];      /* semi-axes (ellipsoids) or sigma (Gaussian) along x,y,z    */
  double arate[3];
} or_prim;

/* Number of trainable parameters P = L(H^2+H)+H+1. */
int64_t or_param_count(int32_t C, int32_t L);

/* eq:rotxsk-rotydk: anticlockwise rotation by theta about (xs0, 0). */
void or_rotate_point(double x, double y, double theta, double xs0, double *xo, double *yo);

/* eq:solvquaddelta/eq:deltaminmax. Returns 0 on miss (disc<0), 1 otherwise,
 * writing the roots clamped to [0,1] (R21). src/dst are (x,y) points. */
int or_fov_delta_bounds(const double src[2], const double dst[2], double xs0, double r,
                        double *dmin, double *dmax);

/* Ray records for n pixels: per sub-ray s (s = v*sub_x + u) 9 doubles
 * {o.x,o.y,o.z, d.x,d.y,d.z, delta_min, delta_max, chord}.  Out: rec[n*S*9].
 * Returns 0, or -1 if an index is out of range (its records are zeroed). */
/* N4 voxel grid: voxel (i,j,k) centre (x0 + (i+1/2) vx, y0 + (j+1/2) vy, z0 + (k+1/2) vz). */
typedef struct {
  int64_t nx, ny, nz;
  double x0, y0, z0;
  double vx, vy, vz;
} or_grid;

/* voxel = pixel / magnification (1 parallel; (sod+odd)/sod fan, cone), grid
 * covering [xs0 - r, xs0 + r] x [-r, r] x [z_lo, z_hi], centred (R25). */
void or_default_grid(const or_geom *g, or_grid *out);

/* mu at the voxel centres of planes [k_begin, k_begin + k_count) at time t:
 * out[((k - k_begin) ny + j) nx + i] = M(normalize(centre, t)), 0 outside the FOV cylinder (R25). */
void or_voxelize(const or_geom *g, const or_field *f, const double *B, const double *params, const or_grid *grid,
                 double t, int64_t k_begin, int64_t k_count, double *out);

/* Philox4x32-10 (Salmon et al. 2011), the counter-based generator of N3: out = bijection of ctr
 * under key.  u01(x) = (x >> 8) 2^-24, exactly representable in fp32 and fp64. */
void or_philox4x32(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* N3 stratified sample offsets: u[(q*S + s)*N_s + j] in [0,1) for pixel idx[q] (0.5 when
 * g->sampling == 0), and the sub-pixel offsets ux, uz of each sub-ray (0.5, 0.5 when off). */
void or_sample_offsets(const or_geom *g, const int64_t *idx, int64_t n, double *u, double *uxz);

int or_rays(const or_geom *g, const double *theta, int64_t M, const int64_t *idx, int64_t n,
            double *rec);

/* GRFF features of n points: out[n*2C] = [cos(2 pi B rbar); sin(2 pi B rbar)]. */
void or_grff(int32_t C, const double *B, const double *rbar, int64_t n, double *out);

/* DINR network M(rbar) = mu0*(w_o.h_L + b_o) at n normalized points rbar[n*4] (t,z,y,x). */
void or_mlp_eval(const or_field *f, const double *B, const double *params, const double *rbar,
                 int64_t n, double *mu_out);
/* grad[P] = sum_j u[j] * dM(rbar_j)/dgamma (reverse mode). */
void or_mlp_grad(const or_field *f, const double *B, const double *params, const double *rbar,
                 const double *u, int64_t n, double *grad);

/* Forward projection (eq:estforwmod + eq:beerstransavg / eq:beersattenavg):
 * fhat[n] (log domain) and optional p_sub[n*S] (per-sub-ray line integrals). */
int or_project(const or_geom *g, const double *theta, const double *t, int64_t M,
               const or_field *f, const double *B, const double *params,
               const int64_t *idx, int64_t n, double *fhat, double *p_sub);

/* Local loss (eq:localoptfunc) and its gradient (eq:partiald, exact chain rule):
 * grad[0..P-1] = dL/dgamma, grad[P] = L. */
int or_project_and_grad(const or_geom *g, const double *theta, const double *t, int64_t M,
                        const or_field *f, const double *B, const double *params,
                        const int64_t *idx, int64_t n, const double *y, double *grad);

/* Same projector with mu given by an analytic phantom (quadrature, O14). mu0 unused. */
int or_project_analytic(const or_geom *g, const double *theta, const double *t, int64_t M,
                        int32_t combine, const or_prim *prims, int32_t n_prims,
                        const int64_t *idx, int64_t n, double *fhat, double *p_sub);

/* Exact line integral of the phantom over delta in [dmin,dmax] of s*mu(o + delta*d)
 * at time t (closed forms; no quadrature). */
double or_line_integral_exact(const or_prim *prims, int32_t n_prims, const double o[3],
                              const double d[3], double dmin, double dmax, double t);

/* Exact per-pixel projection: per sub-ray exact line integrals, then the combine. */
int or_project_exact(const or_geom *g, const double *theta, const double *t, int64_t M,
                     int32_t combine, const or_prim *prims, int32_t n_prims,
                     const int64_t *idx, int64_t n, double *fhat, double *p_sub);

/* Adam ("We use the Adam optimizer"; constants and bias correction as SPEC S:377-383):
 * m <- b1 m + (1-b1) g; v <- b2 v + (1-b2) g^2; param -= lr * mhat / (sqrt(vhat) + eps),
 * mhat = m / (1 - b1^step), vhat = v / (1 - b2^step), step >= 1 (in place, n values). */
void or_adam_step(double *param, const double *grad, double *m, double *v, int64_t n, double lr, double b1,
                  double b2, double eps, int64_t step);

/* N1 sampler ("we randomly choose a subset Omega_k"; epochs P:3333-3336; without
 * replacement via a per-epoch permutation; reading R27 in DESIGN.md).
 * or_perm: the bijection perm_e of [0, D) for epoch e -- an 8-round balanced Feistel network on 2h
 * bits (h >= 1 smallest with 4^h >= D), x = (Lh << h) | Rh, round r: (Lh, Rh) <- (Rh, Lh ^ (F_r(Rh)
 * & (2^h - 1))), F_r(R) = Philox4x32-10(ctr = (R, r, e lo, e hi), key = (seed lo, seed hi ^
 * 0x9E3779B9)) word 0; applied again while the value is >= D (cycle walking). */
int64_t or_perm(int64_t D, uint64_t seed, int64_t epoch, int64_t q);
/* Iteration `it` of epoch `epoch` on process `rank` of `world`, n pixels each (eq:totbatch).
 * mode 0 (view shards): the shard holds views rank, rank + world, ... (nv = ceil((M -
 * rank) / world)), D = nv N; p_j = (it n + j) mod D, q = perm_e(p_j), idx = (rank + world (q / N)) N +
 * q mod N, src = q (the pixel's position in the rank's y shard, stored view by view).
 * mode 1 (one global permutation split contiguously over the processes): D = M N;
 * p_j = (it world n + rank n + j) mod D, idx = src = perm_e(p_j).
 * The last iteration of an epoch wraps to the start of the same permutation, so every process
 * always takes exactly n pixels (R27).  Returns 0, or -1 for bad arguments. */
int or_sample_batch(int64_t M, int64_t N, uint64_t seed, int64_t epoch, int64_t it, int rank, int world, int mode,
                    int64_t n, int64_t *idx, int64_t *src);
/* Iterations per epoch: ceil(M N / (world n)). */
int64_t or_iterations_per_epoch(int64_t M, int64_t N, int world, int64_t n);

/* OpenMP threads the oracle's parallel loops use (omp_get_max_threads; OMP_NUM_THREADS): the
 * "cores" of a host timing of the oracle.  Not part of the method. */
int or_max_threads(void);

#ifdef __cplusplus
}
#endif
#endif
