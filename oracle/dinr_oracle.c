/*
 * dinr_oracle.c -- plain, slow, obviously-correct fp64 CPU ORACLE of the DINR hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see dinr_oracle.h).  Not part of the product; shares no code
 * with paper_2404_19075_b200/csrc.  Build: gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC.
 *
 * Step numbering O1..O14 follows DESIGN.md "Oracle" (= SURVEY.md 8(c)); each step cites the
 * PAPER.md passage it restates.
 */
#include "dinr_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static const double kPi = 3.14159265358979323846;

/* N3: Philox4x32-10, as defined by Salmon, Moraes, Dror, Shaw (SC'11): 10 rounds of
 *   (c0, c1, c2, c3) <- (hi(M1 c2) ^ c1 ^ k0, lo(M1 c2), hi(M0 c0) ^ c3 ^ k1, lo(M0 c0)),
 *   key bumped by the Weyl constants (W0, W1) after every round. */
void or_philox4x32(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3], k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0, n1 = (uint32_t)p1;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1, n3 = (uint32_t)p0;
    c0 = n0;
    c1 = n1;
    c2 = n2;
    c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

static double u01(uint32_t x) { return (double)(x >> 8) * (1.0 / 16777216.0); }

/* uniforms of global ray `ray` (= pixel index * S + s): counter word 0 = j for the sample
 * offsets, 0xFFFFFFFF for the sub-pixel offset pair. */
static void ray_uniforms(const or_geom *g, int64_t ray, uint32_t w0, uint32_t out[4]) {
  uint32_t ctr[4] = {w0, (uint32_t)((uint64_t)ray & 0xFFFFFFFFu), (uint32_t)((uint64_t)ray >> 32), g->step};
  uint32_t key[2] = {(uint32_t)(g->seed & 0xFFFFFFFFu), (uint32_t)(g->seed >> 32)};
  or_philox4x32(ctr, key, out);
}
static double sample_u(const or_geom *g, int64_t ray, int j) {
  if (!g->sampling) return 0.5; /* R8 midpoint */
  uint32_t o[4];
  ray_uniforms(g, ray, (uint32_t)j, o);
  return u01(o[0]);
}
static void subpixel_u(const or_geom *g, int64_t ray, double *ux, double *uz) {
  if (!g->sampling) {
    *ux = 0.5;
    *uz = 0.5;
    return;
  }
  uint32_t o[4];
  ray_uniforms(g, ray, 0xFFFFFFFFu, o);
  *ux = u01(o[0]);
  *uz = u01(o[1]);
}

int64_t or_param_count(int32_t C, int32_t L) {
  /* L FC layers 2C->2C with bias, head 2C->1 with bias. */
  int64_t H = 2 * (int64_t)C;
  return (int64_t)L * (H * H + H) + H + 1;
}

/* O4, eq:rotxsk / eq:rotysk, exact operation order:
 *   x' = (x cos - y sin) + (xs0 - xs0 cos),  y' = (x sin + y cos) - xs0 sin. */
static void rotate_cs(double x, double y, double c, double s, double xs0, double *xo, double *yo) {
  *xo = (x * c - y * s) + (xs0 - xs0 * c);
  *yo = (x * s + y * c) - xs0 * s;
}

void or_rotate_point(double x, double y, double theta, double xs0, double *xo, double *yo) {
  rotate_cs(x, y, cos(theta), sin(theta), xs0, xo, yo); /* O1: host libm cos/sin */
}

/* O3, eq:solvquaddelta / eq:deltaminmax, with the FOV cylinder
 * (x - xs0)^2 + y^2 <= r^2.  a,b,c as printed at P:2830-2833. */
static int delta_bounds(double xs, double ys, double xd, double yd, double xs0, double r,
                        double *a_out, double *dmin, double *dmax) {
  double ex = xd - xs, ey = yd - ys, px = xs - xs0;
  double a = ex * ex + ey * ey;
  double b = 2.0 * (px * ex + ys * ey);
  double c = (px * px + ys * ys) - r * r;
  double disc = b * b - 4.0 * a * c;
  *a_out = a;
  if (disc < 0.0) { /* R21: miss */
    *dmin = 0.0;
    *dmax = 0.0;
    return 0;
  }
  double q = sqrt(disc);
  double lo = (-b - q) / (2.0 * a);
  double hi = (-b + q) / (2.0 * a);
  *dmin = fmin(fmax(lo, 0.0), 1.0);
  *dmax = fmin(fmax(hi, 0.0), 1.0);
  return 1;
}

int or_fov_delta_bounds(const double src[2], const double dst[2], double xs0, double r,
                        double *dmin, double *dmax) {
  double a;
  return delta_bounds(src[0], src[1], dst[0], dst[1], xs0, r, &a, dmin, dmax);
}

/* O2 (P:53-69 pixel area C_ij; P:366-374 D x D sub-pixel centres; P:2842-2853 cone source;
 * R9 fan, R10 parallel), O3 (bounds, theta-invariant P:2812-2818), A5 arc length
 * (P:155-172 read as the Euclidean norm, R1), O4 rotation. */
static void ray_record(const or_geom *g, double ck, double sk, int64_t row, int64_t col, int u,
                       int v, double ux, double uz, double rec[9]) {
  /* sub-pixel (u, v) at offset (ux, uz) in its cell: 1/2 = centre (midpoint, R8), N3 jitter */
  double xd = -g->cx + ((double)col + ((double)u + ux) / (double)g->sub_x) * g->dx;
  double yd = g->odd;
  double zd = -g->cz + ((double)row + ((double)v + uz) / (double)g->sub_z) * g->dz;
  double xs, ys = -g->sod, zs;
  if (g->beam == 2) {        /* cone: point source (0,-SOD,0) */
    xs = 0.0;
    zs = 0.0;
  } else if (g->beam == 1) { /* fan: (0,-SOD,z_d), R9 */
    xs = 0.0;
    zs = zd;
  } else {                   /* parallel: (x_d,-SOD,z_d), R10 */
    xs = xd;
    zs = zd;
  }
  double a, dmin, dmax;
  delta_bounds(xs, ys, xd, yd, g->xs0, g->r, &a, &dmin, &dmax);
  double ez = zd - zs;
  double s = sqrt(a + ez * ez);
  double chord = s * (dmax - dmin);
  double xsk, ysk, xdk, ydk;
  rotate_cs(xs, ys, ck, sk, g->xs0, &xsk, &ysk);
  rotate_cs(xd, yd, ck, sk, g->xs0, &xdk, &ydk);
  rec[0] = xsk;
  rec[1] = ysk;
  rec[2] = zs;
  rec[3] = xdk - xsk;
  rec[4] = ydk - ysk;
  rec[5] = zd - zs;
  rec[6] = dmin;
  rec[7] = dmax;
  rec[8] = chord;
}

/* all S sub-rays of pixel i (global index), s = v * sub_x + u */
static void pixel_rays(const or_geom *g, double ck, double sk, int64_t i, int64_t row, int64_t col, double *rec) {
  int S = g->sub_x * g->sub_z;
  for (int v = 0; v < g->sub_z; ++v)
    for (int u = 0; u < g->sub_x; ++u) {
      int s = v * g->sub_x + u;
      double ux, uz;
      subpixel_u(g, i * S + s, &ux, &uz);
      ray_record(g, ck, sk, row, col, u, v, ux, uz, rec + s * 9);
    }
}

/* a1 (R13): i = mN + n -> view k, detector pixel n = row*n_cols + col. */
static int decode(const or_geom *g, int64_t M, int64_t i, int64_t *k, int64_t *row, int64_t *col) {
  int64_t N = (int64_t)g->n_rows * g->n_cols;
  if (i < 0 || i >= M * N) return -1;
  *k = i / N;
  int64_t n = i % N;
  *row = n / g->n_cols;
  *col = n % g->n_cols;
  return 0;
}

void or_sample_offsets(const or_geom *g, const int64_t *idx, int64_t n, double *u, double *uxz) {
  int S = g->sub_x * g->sub_z, ns = g->n_s;
  for (int64_t q = 0; q < n; ++q)
    for (int s = 0; s < S; ++s) {
      int64_t ray = idx[q] * S + s;
      if (u)
        for (int j = 0; j < ns; ++j) u[(q * S + s) * ns + j] = sample_u(g, ray, j);
      if (uxz) subpixel_u(g, ray, uxz + (q * S + s) * 2, uxz + (q * S + s) * 2 + 1);
    }
}

int or_rays(const or_geom *g, const double *theta, int64_t M, const int64_t *idx, int64_t n,
            double *rec) {
  int S = g->sub_x * g->sub_z;
  int err = 0;
  for (int64_t p = 0; p < n; ++p) {
    int64_t k, row, col;
    double *out = rec + p * S * 9;
    if (decode(g, M, idx[p], &k, &row, &col)) {
      memset(out, 0, sizeof(double) * 9 * S);
      err = -1;
      continue;
    }
    double ck = cos(theta[k]), sk = sin(theta[k]); /* O1 */
    pixel_rays(g, ck, sk, idx[p], row, col, out);
  }
  return err;
}

/* ---------------------------------------------------------------------------------------
 * Field network.  Parameter layout (D5): for l=1..L: W_l (H x H, [out][in]),
 * b_l (H); then w_o (H), b_o.
 * ------------------------------------------------------------------------------------- */
typedef struct {
  int C, L, H;
  const double *B, *prm;
  double mu0;
} net_t;

static net_t make_net(const or_field *f, const double *B, const double *prm) {
  net_t n;
  n.C = f->C;
  n.L = f->L;
  n.H = 2 * f->C;
  n.B = B;
  n.prm = prm;
  n.mu0 = f->mu0;
  return n;
}

/* O7 GRFF: phi_c = sum_q B[c][q] rbar_q; [cos(2 pi phi) ; sin(2 pi phi)]. */
static void grff(const net_t *nt, const double rb[4], double *h0) {
  for (int c = 0; c < nt->C; ++c) {
    double phi = 0.0;
    for (int q = 0; q < 4; ++q) phi += nt->B[c * 4 + q] * rb[q];
    h0[c] = cos(2.0 * kPi * phi);
    h0[nt->C + c] = sin(2.0 * kPi * phi);
  }
}

void or_grff(int32_t C, const double *B, const double *rbar, int64_t n, double *out) {
  net_t nt;
  nt.C = C;
  nt.B = B;
  for (int64_t j = 0; j < n; ++j) grff(&nt, rbar + 4 * j, out + j * 2 * C);
}

static double sigmoid(double z) { return 1.0 / (1.0 + exp(-z)); }

/* O8: z_l = W_l h_{l-1} + b_l, h_l = swish(z_l) = z sigma(z) (R19, beta=1);
 * returns M = mu0 * (w_o . h_L + b_o) (R6: mu0 applied once).  hs[(L+1)*H], zs[L*H]. */
static double mlp_forward(const net_t *nt, const double rb[4], double *hs, double *zs) {
  int H = nt->H;
  grff(nt, rb, hs);
  for (int l = 0; l < nt->L; ++l) {
    const double *W = nt->prm + (int64_t)l * (H * H + H);
    const double *b = W + (int64_t)H * H;
    const double *hin = hs + (int64_t)l * H;
    double *z = zs + (int64_t)l * H, *hout = hs + (int64_t)(l + 1) * H;
    for (int o = 0; o < H; ++o) {
      double acc = 0.0;
      for (int i = 0; i < H; ++i) acc += W[(int64_t)o * H + i] * hin[i];
      z[o] = acc + b[o];
      hout[o] = z[o] * sigmoid(z[o]);
    }
  }
  const double *wo = nt->prm + (int64_t)nt->L * (H * H + H);
  double raw = 0.0;
  const double *hL = hs + (int64_t)nt->L * H;
  for (int i = 0; i < H; ++i) raw += wo[i] * hL[i];
  raw += wo[H];
  return nt->mu0 * raw;
}

/* O12: reverse mode of M for one sample with upstream u = dLoss/dM, accumulated into grad.
 * swish'(z) = sigma (1 + z (1 - sigma)); e_{l-1} = W_l^T delta_l. */
static void mlp_backward(const net_t *nt, const double *hs, const double *zs, double u, double *grad,
                         double *e, double *enew) {
  int H = nt->H, L = nt->L;
  int64_t off_o = (int64_t)L * (H * H + H);
  const double *wo = nt->prm + off_o;
  const double *hL = hs + (int64_t)L * H;
  double ur = u * nt->mu0;
  grad[off_o + H] += ur;
  for (int i = 0; i < H; ++i) {
    grad[off_o + i] += ur * hL[i];
    e[i] = ur * wo[i];
  }
  for (int l = L - 1; l >= 0; --l) {
    const double *W = nt->prm + (int64_t)l * (H * H + H);
    double *gW = grad + (int64_t)l * (H * H + H);
    double *gb = gW + (int64_t)H * H;
    const double *z = zs + (int64_t)l * H, *hin = hs + (int64_t)l * H;
    for (int o = 0; o < H; ++o) {
      double sg = sigmoid(z[o]);
      e[o] = e[o] * (sg * (1.0 + z[o] * (1.0 - sg))); /* delta_l */
    }
    for (int o = 0; o < H; ++o) {
      double dl = e[o];
      gb[o] += dl;
      for (int i = 0; i < H; ++i) gW[(int64_t)o * H + i] += dl * hin[i];
    }
    if (l > 0) {
      for (int i = 0; i < H; ++i) {
        double acc = 0.0;
        for (int o = 0; o < H; ++o) acc += W[(int64_t)o * H + i] * e[o];
        enew[i] = acc;
      }
      memcpy(e, enew, sizeof(double) * H);
    }
  }
}

void or_mlp_eval(const or_field *f, const double *B, const double *params, const double *rbar,
                 int64_t n, double *mu_out) {
  net_t nt = make_net(f, B, params);
#pragma omp parallel
  {
    double *hs = (double *)malloc(sizeof(double) * (size_t)(nt.L + 1) * nt.H);
    double *zs = (double *)malloc(sizeof(double) * (size_t)nt.L * nt.H);
#pragma omp for schedule(static)
    for (int64_t j = 0; j < n; ++j) mu_out[j] = mlp_forward(&nt, rbar + 4 * j, hs, zs);
    free(hs);
    free(zs);
  }
}

void or_mlp_grad(const or_field *f, const double *B, const double *params, const double *rbar,
                 const double *u, int64_t n, double *grad) {
  net_t nt = make_net(f, B, params);
  int64_t P = or_param_count(f->C, f->L);
  memset(grad, 0, sizeof(double) * P);
  double *hs = (double *)malloc(sizeof(double) * (size_t)(nt.L + 1) * nt.H);
  double *zs = (double *)malloc(sizeof(double) * (size_t)nt.L * nt.H);
  double *e = (double *)malloc(sizeof(double) * nt.H), *en = (double *)malloc(sizeof(double) * nt.H);
  for (int64_t j = 0; j < n; ++j) {
    mlp_forward(&nt, rbar + 4 * j, hs, zs);
    mlp_backward(&nt, hs, zs, u[j], grad, e, en);
  }
  free(hs);
  free(zs);
  free(e);
  free(en);
}

/* O6 normalization (R11 explicit box, R12 order (t,z,y,x)). */
static void normalize(const or_geom *g, double x, double y, double z, double t, double rb[4]) {
  double ct = 0.5 * (g->t_lo + g->t_hi), ht = 0.5 * (g->t_hi - g->t_lo);
  double cz = 0.5 * (g->z_lo + g->z_hi), hz = 0.5 * (g->z_hi - g->z_lo);
  rb[0] = ht > 0.0 ? (t - ct) / ht : 0.0;
  rb[1] = hz > 0.0 ? (z - cz) / hz : 0.0;
  rb[2] = y / g->r;
  rb[3] = (x - g->xs0) / g->r;
}

/* O5: samples delta_j = dmin + (j + u_j) (dmax - dmin)/N_s, X_j = o + delta_j d; u_j = 1/2 is
 * the midpoint rule (R8), u_j ~ U[0,1) the stratified jitter of N3 (eq:estforwmod). */
static void sample_point(const double rec[9], int ns, int j, double uj, double X[3]) {
  double step = (rec[7] - rec[6]) / (double)ns;
  double dj = rec[6] + ((double)j + uj) * step;
  X[0] = rec[0] + dj * rec[3];
  X[1] = rec[1] + dj * rec[4];
  X[2] = rec[2] + dj * rec[5];
}

/* O10 (eq:beerstransavg P:184-203 / eq:beersattenavg P:204-256; R5, R22):
 *   BEER:   fhat = -log( (1/S) sum_s exp(-p_s) ) computed as m - log((1/S) sum exp(-(p_s - m)))
 *   LINEAR: fhat = (1/S) sum_s p_s.
 * pi[s] = d fhat / d p_s. */
static double combine(int mode, const double *p, int S, double *pi) {
  if (mode == 1) {
    double acc = 0.0;
    for (int s = 0; s < S; ++s) acc += p[s];
    if (pi)
      for (int s = 0; s < S; ++s) pi[s] = 1.0 / (double)S;
    return acc / (double)S;
  }
  double m = p[0];
  for (int s = 1; s < S; ++s) m = fmin(m, p[s]);
  double T = 0.0;
  for (int s = 0; s < S; ++s) T += exp(-(p[s] - m));
  T /= (double)S;
  if (pi)
    for (int s = 0; s < S; ++s) pi[s] = exp(-(p[s] - m)) / ((double)S * T);
  return m - log(T);
}

/* Per-pixel forward with the network; optionally stores activations for the backward. */
typedef struct {
  double *hs, *zs; /* [S*Ns][(L+1)H], [S*Ns][LH] */
  double *rec;     /* S*9 */
  double *p;       /* S */
  double *pi;      /* S */
  double *e, *en;
} pix_ws;

static int pixel_forward(const or_geom *g, const double *theta, const double *t, int64_t M,
                         const net_t *nt, int combine_mode, int64_t i, pix_ws *w, int store,
                         double *fhat) {
  int S = g->sub_x * g->sub_z, ns = g->n_s, H = nt->H, L = nt->L;
  int64_t k, row, col;
  if (decode(g, M, i, &k, &row, &col)) {
    for (int s = 0; s < S; ++s) w->p[s] = 0.0;
    *fhat = 0.0;
    return -1;
  }
  double ck = cos(theta[k]), sk = sin(theta[k]);
  pixel_rays(g, ck, sk, i, row, col, w->rec);
  for (int s = 0; s < S; ++s) {
    const double *rec = w->rec + s * 9;
    double sum = 0.0;
    if (rec[8] > 0.0) { /* R21: a ray contributes iff its chord is positive */
      for (int j = 0; j < ns; ++j) {
        double X[3], rb[4];
        sample_point(rec, ns, j, sample_u(g, i * S + s, j), X);
        normalize(g, X[0], X[1], X[2], t[k], rb);
        int64_t sj = (int64_t)s * ns + j;
        double *hs = w->hs + (store ? sj * (int64_t)(L + 1) * H : 0);
        double *zs = w->zs + (store ? sj * (int64_t)L * H : 0);
        sum += mlp_forward(nt, rb, hs, zs);
      }
    }
    /* O9, eq:estforwmod with R7: p_s = (chord/N_s) sum_j mu_j */
    w->p[s] = rec[8] > 0.0 ? (rec[8] / (double)ns) * sum : 0.0;
  }
  *fhat = combine(combine_mode, w->p, S, w->pi);
  return 0;
}

static pix_ws ws_alloc(int S, int ns, int H, int L, int store) {
  pix_ws w;
  size_t nsamp = store ? (size_t)S * ns : 1;
  w.hs = (double *)malloc(sizeof(double) * nsamp * (L + 1) * H);
  w.zs = (double *)malloc(sizeof(double) * nsamp * L * H);
  w.rec = (double *)malloc(sizeof(double) * S * 9);
  w.p = (double *)malloc(sizeof(double) * S);
  w.pi = (double *)malloc(sizeof(double) * S);
  w.e = (double *)malloc(sizeof(double) * H);
  w.en = (double *)malloc(sizeof(double) * H);
  return w;
}

static void ws_free(pix_ws *w) {
  free(w->hs);
  free(w->zs);
  free(w->rec);
  free(w->p);
  free(w->pi);
  free(w->e);
  free(w->en);
}

int or_project(const or_geom *g, const double *theta, const double *t, int64_t M,
               const or_field *f, const double *B, const double *params,
               const int64_t *idx, int64_t n, double *fhat, double *p_sub) {
  net_t nt = make_net(f, B, params);
  int S = g->sub_x * g->sub_z;
  int err = 0;
#pragma omp parallel reduction(| : err)
  {
    pix_ws w = ws_alloc(S, g->n_s, nt.H, nt.L, 0);
#pragma omp for schedule(dynamic, 1)
    for (int64_t p = 0; p < n; ++p) {
      err |= pixel_forward(g, theta, t, M, &nt, f->combine, idx[p], &w, 0, &fhat[p]) ? 1 : 0;
      if (p_sub)
        for (int s = 0; s < S; ++s) p_sub[p * S + s] = w.p[s];
    }
    ws_free(&w);
  }
  return err ? -1 : 0;
}

/* eq:mainsqdist / eq:localoptfunc: L = (1/n) sum_i (y_i - fhat_i)^2;
 * gradient by the chain rule (eq:partiald P:414-420, revised form, R15):
 *   g_i = dL/dfhat_i = -2 (y_i - fhat_i)/n,  dfhat/dp_s = pi_s,  dp_s/dM_j = chord_s/N_s. */
int or_project_and_grad(const or_geom *g, const double *theta, const double *t, int64_t M,
                        const or_field *f, const double *B, const double *params,
                        const int64_t *idx, int64_t n, const double *y, double *grad) {
  net_t nt = make_net(f, B, params);
  int S = g->sub_x * g->sub_z, ns = g->n_s, H = nt.H, L = nt.L;
  int64_t P = or_param_count(f->C, f->L);
  memset(grad, 0, sizeof(double) * (P + 1));
  if (n == 0) return 0;
  int nthr = 1;
#ifdef _OPENMP
  nthr = omp_get_max_threads();
#endif
  double *part = (double *)calloc((size_t)nthr * (P + 1), sizeof(double));
  int err = 0;
#pragma omp parallel num_threads(nthr) reduction(| : err)
  {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
    double *gacc = part + (size_t)tid * (P + 1);
    pix_ws w = ws_alloc(S, ns, H, L, 1);
#pragma omp for schedule(static)
    for (int64_t p = 0; p < n; ++p) {
      double fh;
      err |= pixel_forward(g, theta, t, M, &nt, f->combine, idx[p], &w, 1, &fh) ? 1 : 0;
      double r = y[p] - fh;
      gacc[P] += r * r;
      double gi = -2.0 * r / (double)n;
      for (int s = 0; s < S; ++s) {
        const double *rec = w.rec + s * 9;
        if (!(rec[8] > 0.0)) continue;
        double us = gi * w.pi[s] * (rec[8] / (double)ns);
        for (int j = 0; j < ns; ++j) {
          int64_t sj = (int64_t)s * ns + j;
          mlp_backward(&nt, w.hs + sj * (int64_t)(L + 1) * H, w.zs + sj * (int64_t)L * H, us, gacc, w.e, w.en);
        }
      }
    }
    ws_free(&w);
  }
  for (int th = 0; th < nthr; ++th)
    for (int64_t q = 0; q <= P; ++q) grad[q] += part[(size_t)th * (P + 1) + q];
  grad[P] /= (double)n;
  free(part);
  return err ? -1 : 0;
}

/* ---------------------------------------------------------------------------------------
 * Analytic phantoms (O14): point evaluation and exact line integrals.
 * ------------------------------------------------------------------------------------- */
static void prim_state(const or_prim *q, double t, double c[3], double a[3]) {
  for (int k = 0; k < 3; ++k) {
    c[k] = q->c0[k] + q->vel[k] * t;
    a[k] = q->a0[k] + q->arate[k] * t;
  }
}

static double phantom_mu(const or_prim *prims, int np, const double X[3], double t) {
  double mu = 0.0;
  for (int q = 0; q < np; ++q) {
    double c[3], a[3], rho2 = 0.0;
    prim_state(&prims[q], t, c, a);
    for (int k = 0; k < 3; ++k) {
      double u = (X[k] - c[k]) / a[k];
      rho2 += u * u;
    }
    if (prims[q].kind == 0) {
      if (rho2 <= 1.0) mu += prims[q].value;
    } else if (prims[q].kind == 1) {
      if (rho2 <= 1.0) mu += prims[q].value * (1.0 - rho2) * (1.0 - rho2);
    } else {
      mu += prims[q].value * exp(-0.5 * rho2);
    }
  }
  return mu;
}

/* Closed forms (SURVEY 8(c) "Closed forms for the phantom pins"), in the delta
 * parameterization: rho^2(delta) = A delta^2 + Bq delta + Cq. */
double or_line_integral_exact(const or_prim *prims, int32_t n_prims, const double o[3],
                              const double d[3], double dmin, double dmax, double t) {
  double s = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
  double total = 0.0;
  if (!(dmax > dmin)) return 0.0;
  for (int q = 0; q < n_prims; ++q) {
    double c[3], a[3], A = 0.0, Bq = 0.0, Cq = 0.0;
    prim_state(&prims[q], t, c, a);
    for (int k = 0; k < 3; ++k) {
      double dk = d[k] / a[k], ok = (o[k] - c[k]) / a[k];
      A += dk * dk;
      Bq += 2.0 * ok * dk;
      Cq += ok * ok;
    }
    double dc = -Bq / (2.0 * A);
    double rmin2 = Cq - Bq * Bq / (4.0 * A); /* rho^2 at the closest point */
    if (prims[q].kind == 2) {
      /* integral of A exp(-rho^2/2) over [dmin,dmax] (erf form, tails via erfc) */
      double k2 = sqrt(0.5 * A);
      double x1 = k2 * (dmin - dc), x2 = k2 * (dmax - dc), diff;
      if (x1 >= 0.0)
        diff = erfc(x1) - erfc(x2);
      else if (x2 <= 0.0)
        diff = erfc(-x2) - erfc(-x1);
      else
        diff = erf(x2) - erf(x1);
      total += s * prims[q].value * exp(-0.5 * rmin2) * sqrt(kPi / (2.0 * A)) * diff;
      continue;
    }
    if (rmin2 >= 1.0) continue; /* misses (or grazes) the ellipsoid */
    double h = sqrt((1.0 - rmin2) / A);
    double lo = fmax(dc - h, dmin) - dc, hi = fmin(dc + h, dmax) - dc;
    if (!(hi > lo)) continue;
    if (prims[q].kind == 0) {
      total += s * prims[q].value * (hi - lo);
    } else {
      /* mu_c (1 - rho^2)^2 = mu_c A^2 (h^2 - u^2)^2; antiderivative h^4 u - 2/3 h^2 u^3 + u^5/5 */
      double h2 = h * h;
#define F_POLY(u) (h2 * h2 * (u) - (2.0 / 3.0) * h2 * (u) * (u) * (u) + (u) * (u) * (u) * (u) * (u) / 5.0)
      total += s * prims[q].value * A * A * (F_POLY(hi) - F_POLY(lo));
#undef F_POLY
    }
  }
  return total;
}

int or_project_analytic(const or_geom *g, const double *theta, const double *t, int64_t M,
                        int32_t combine_mode, const or_prim *prims, int32_t n_prims,
                        const int64_t *idx, int64_t n, double *fhat, double *p_sub) {
  int S = g->sub_x * g->sub_z, ns = g->n_s;
  int err = 0;
#pragma omp parallel reduction(| : err)
  {
    double *rec = (double *)malloc(sizeof(double) * S * 9), *p = (double *)malloc(sizeof(double) * S);
#pragma omp for schedule(dynamic, 4)
    for (int64_t q = 0; q < n; ++q) {
      int64_t k, row, col;
      if (decode(g, M, idx[q], &k, &row, &col)) {
        err |= 1;
        for (int s = 0; s < S; ++s) p[s] = 0.0;
      } else {
        double ck = cos(theta[k]), sk = sin(theta[k]);
        pixel_rays(g, ck, sk, idx[q], row, col, rec);
        for (int s = 0; s < S; ++s) {
          double sum = 0.0;
          if (rec[s * 9 + 8] > 0.0)
            for (int j = 0; j < ns; ++j) {
              double X[3];
              sample_point(rec + s * 9, ns, j, sample_u(g, idx[q] * S + s, j), X);
              sum += phantom_mu(prims, n_prims, X, t[k]);
            }
          p[s] = rec[s * 9 + 8] > 0.0 ? (rec[s * 9 + 8] / (double)ns) * sum : 0.0;
        }
      }
      fhat[q] = combine(combine_mode, p, S, NULL);
      if (p_sub)
        for (int s = 0; s < S; ++s) p_sub[q * S + s] = p[s];
    }
    free(rec);
    free(p);
  }
  return err ? -1 : 0;
}

int or_project_exact(const or_geom *g, const double *theta, const double *t, int64_t M,
                     int32_t combine_mode, const or_prim *prims, int32_t n_prims,
                     const int64_t *idx, int64_t n, double *fhat, double *p_sub) {
  int S = g->sub_x * g->sub_z;
  int err = 0;
#pragma omp parallel reduction(| : err)
  {
    double *rec = (double *)malloc(sizeof(double) * S * 9), *p = (double *)malloc(sizeof(double) * S);
#pragma omp for schedule(dynamic, 16)
    for (int64_t q = 0; q < n; ++q) {
      int64_t k, row, col;
      if (decode(g, M, idx[q], &k, &row, &col)) {
        err |= 1;
        for (int s = 0; s < S; ++s) p[s] = 0.0;
      } else {
        double ck = cos(theta[k]), sk = sin(theta[k]);
        pixel_rays(g, ck, sk, idx[q], row, col, rec);
        for (int s = 0; s < S; ++s) {
          const double *r = rec + s * 9;
          p[s] = r[8] > 0.0 ? or_line_integral_exact(prims, n_prims, r, r + 3, r[6], r[7], t[k]) : 0.0;
        }
      }
      fhat[q] = combine(combine_mode, p, S, NULL);
      if (p_sub)
        for (int s = 0; s < S; ++s) p_sub[q * S + s] = p[s];
    }
    free(rec);
    free(p);
  }
  return err ? -1 : 0;
}

/* N4 ------------------------------------------------------------ */
void or_default_grid(const or_geom *g, or_grid *out) {
  /* "a spatial resolution equal to the detector pixel size divided by the geometric
   * magnification ... one for parallel-beam and ... the ratio of the source-to-detector
   * distance and the source-to-object distance for cone-beam" */
  double mag = g->beam == 0 ? 1.0 : (g->sod + g->odd) / g->sod;
  double vx = g->dx / mag, vz = g->dz / mag;
  out->vx = vx;
  out->vy = vx;
  out->vz = vz;
  out->nx = (int64_t)ceil(2.0 * g->r / vx);
  out->ny = out->nx;
  out->nz = (int64_t)ceil((g->z_hi - g->z_lo) / vz);
  if (out->nz < 1) out->nz = 1;
  out->x0 = g->xs0 - 0.5 * (double)out->nx * vx;
  out->y0 = -0.5 * (double)out->ny * vx;
  out->z0 = 0.5 * (g->z_lo + g->z_hi) - 0.5 * (double)out->nz * vz;
}

void or_voxelize(const or_geom *g, const or_field *f, const double *B, const double *params, const or_grid *grid,
                 double t, int64_t k_begin, int64_t k_count, double *out) {
  net_t nt = make_net(f, B, params);
  int64_t plane = grid->nx * grid->ny, n = plane * k_count;
#pragma omp parallel
  {
    double *hs = (double *)malloc(sizeof(double) * (size_t)(nt.L + 1) * nt.H);
    double *zs = (double *)malloc(sizeof(double) * (size_t)nt.L * nt.H);
#pragma omp for schedule(static)
    for (int64_t v = 0; v < n; ++v) {
      int64_t i = v % grid->nx, j = (v / grid->nx) % grid->ny, k = k_begin + v / plane;
      double x = grid->x0 + ((double)i + 0.5) * grid->vx;
      double y = grid->y0 + ((double)j + 0.5) * grid->vy;
      double z = grid->z0 + ((double)k + 0.5) * grid->vz;
      double px = x - g->xs0;
      if (px * px + y * y <= g->r * g->r) { /* FOV cylinder, R25 */
        double rb[4];
        normalize(g, x, y, z, t, rb);
        out[v] = mlp_forward(&nt, rb, hs, zs);
      } else {
        out[v] = 0.0;
      }
    }
    free(hs);
    free(zs);
  }
}

void or_adam_step(double *param, const double *grad, double *m, double *v, int64_t n, double lr, double b1,
                  double b2, double eps, int64_t step) {
  double c1 = 1.0 - pow(b1, (double)step), c2 = 1.0 - pow(b2, (double)step);
  for (int64_t q = 0; q < n; ++q) {
    m[q] = b1 * m[q] + (1.0 - b1) * grad[q];
    v[q] = b2 * v[q] + (1.0 - b2) * grad[q] * grad[q];
    double mh = m[q] / c1, vh = v[q] / c2;
    param[q] -= lr * mh / (sqrt(vh) + eps);
  }
}

/* ---------------------------------------------------------------- N1 sampler (R27) */
int64_t or_perm(int64_t D, uint64_t seed, int64_t epoch, int64_t q) {
  int h = 1;
  while (((uint64_t)1 << (2 * h)) < (uint64_t)D) ++h;
  const uint64_t mask = ((uint64_t)1 << h) - 1;
  const uint32_t key[2] = {(uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32) ^ 0x9E3779B9u};
  uint64_t x = (uint64_t)q;
  do {
    uint64_t lh = x >> h, rh = x & mask;
    for (uint32_t r = 0; r < 8; ++r) {
      uint32_t ctr[4] = {(uint32_t)rh, r, (uint32_t)((uint64_t)epoch & 0xFFFFFFFFu), (uint32_t)((uint64_t)epoch >> 32)};
      uint32_t out[4];
      or_philox4x32(ctr, key, out);
      uint64_t nl = rh, nr = lh ^ ((uint64_t)out[0] & mask);
      lh = nl;
      rh = nr;
    }
    x = (lh << h) | rh;
  } while (x >= (uint64_t)D);
  return (int64_t)x;
}

int64_t or_iterations_per_epoch(int64_t M, int64_t N, int world, int64_t n) {
  const int64_t per = (int64_t)world * n;
  return (M * N + per - 1) / per;
}

int or_sample_batch(int64_t M, int64_t N, uint64_t seed, int64_t epoch, int64_t it, int rank, int world, int mode,
                    int64_t n, int64_t *idx, int64_t *src) {
  if (M < 1 || N < 1 || world < 1 || rank < 0 || rank >= world || n < 0 || epoch < 0 || it < 0) return -1;
  if (mode == 0) {
    const int64_t nv = (M - rank + world - 1) / world;
    if (nv < 1) return -1;
    const int64_t D = nv * N;
    for (int64_t j = 0; j < n; ++j) {
      const int64_t p = (it * n + j) % D;
      const int64_t q = or_perm(D, seed, epoch, p);
      const int64_t view = rank + (int64_t)world * (q / N);
      idx[j] = view * N + q % N;
      src[j] = q;
    }
  } else if (mode == 1) {
    const int64_t D = M * N;
    for (int64_t j = 0; j < n; ++j) {
      const int64_t p = (it * world * n + (int64_t)rank * n + j) % D;
      idx[j] = src[j] = or_perm(D, seed, epoch, p);
    }
  } else {
    return -1;
  }
  return 0;
}

int or_max_threads(void) { return omp_get_max_threads(); }
