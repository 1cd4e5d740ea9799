/*
 * dinr.h -- C ABI of libdinr.so, the B200 (sm_100a) differentiable forward projector of
 * arXiv 2404.19075 (DINR, "Distributed Stochastic Optimization of a Neural Representation
 * Network for Time-Space Tomography Reconstruction").
 *
 * Citations: "P:n" = line n of PAPER.md (paper text), "S:n" = line n of SPEC.md,
 * "R#" = reading # in DESIGN.md ("Readings of the paper").  Everything below is plain C:
 * pointers, sizes and status codes.  No C++ exception crosses this boundary.
 *
 * Ownership and threading:
 *   - The caller owns every buffer passed in (device "_dev" buffers and host buffers) and
 *     the CUDA stream; all device work is enqueued on that stream (stream-ordered, async)
 *     unless a function says it synchronizes.
 *   - The context owns the per-view table, packed bf16 weights, scratch (ray records,
 *     per-chunk ray sums, upstream gradients, activation stashes, gradient partials),
 *     timing events and the NCCL communicator.  One context per device per process; a
 *     context is not thread-safe (serialize calls on it), and its calls must be ordered on
 *     one stream (or synchronized between streams): consecutive calls reuse the same scratch.
 *   - Scratch grows on demand with the largest n seen.  Growth allocates; pre-size it with
 *     one untimed call before capturing a CUDA graph.
 * Errors:
 *   - Host-checkable violations return DINR_EINVAL with no side effects.
 *   - Out-of-range pixel indices (i >= M*N) are seen only on the device: they set a sticky
 *     device flag, the pixel contributes 0 (fhat = 0, zero gradient), and
 *     dinr_get_device_status() later returns DINR_ERANGE.
 *   - A ray that misses the FOV is not an error: p_s = 0 and zero gradient (R21).
 *   - CUDA / NCCL failures return DINR_ECUDA / DINR_ENCCL; dinr_last_error() has the text.
 */
#ifndef DINR_H
#define DINR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dinr_ctx dinr_ctx; /* opaque */

typedef enum {
  DINR_OK = 0,
  DINR_EINVAL = 1,  /* invalid argument (host-checked, no side effects)          */
  DINR_ERANGE = 2,  /* a pixel index was out of range (sticky device flag)        */
  DINR_ENOMEM = 3,  /* device allocation failed                                   */
  DINR_ECUDA = 4,   /* CUDA runtime error                                         */
  DINR_ENCCL = 5,   /* NCCL error                                                 */
  DINR_ESTATE = 6,  /* call order violated (e.g. weights before geometry)         */
  DINR_EDEVICE = 7  /* device is not an sm_100 part                               */
} dinr_status;

typedef enum { DINR_PARALLEL = 0, DINR_FAN = 1, DINR_CONE = 2 } dinr_beam;

/* Sub-ray combine: BEER = per-sub-ray Beer's law averaged over the pixel in transmission
 * (eq:beerstransavg; default, north_star); LINEAR = average of the line
 * integrals (eq:beersattenavg / eq:forwmodproj). R5. */
typedef enum { DINR_BEER = 0, DINR_LINEAR = 1 } dinr_combine;

/* BF16: tcgen05 tensor-core MLP (bf16 operands, fp32 accumulate, fp32 epilogue/head).
 * FP32_VERIFY: fp32 CUDA-core MLP with accurate sin/cos/exp (the 1e-5 verification mode). */
typedef enum { DINR_BF16 = 0, DINR_FP32_VERIFY = 1 } dinr_precision;

/* Sample placement (N3): MIDPOINT = sub-pixel centres and sample j at (j + 1/2)/N_s of the FOV
 * chord (R8); JITTER = stratified jitter, the sub-ray at a uniform point of its sub-pixel cell
 * and sample j at (j + u_j)/N_s, uniforms from Philox4x32-10 ("randomly sampled
 * coordinates", eq:estforwmod). */
typedef enum { DINR_MIDPOINT = 0, DINR_JITTER = 1 } dinr_sampling;

/* Scanner geometry (all lengths in one unit, e.g. mm; fp64).
 *   Detector pixel (row j, col i) covers x_d in [-C_x + i*dx, -C_x + (i+1)*dx),
 *   z_d in [-C_z + j*dz, -C_z + (j+1)*dz) on the plane y = +odd.
 *   Sources: cone (0,-sod,0); fan (0,-sod,z_d) (R9); parallel (x_d,-sod,z_d) (R10).
 *   sub_x x sub_z sub-pixel rays to sub-pixel centres, sub-ray s = v*sub_x + u.
 *   FOV: cylinder (x - rot_center_x)^2 + y^2 <= fov_radius^2, infinite in z.
 *   samples_per_ray N_s: fixed midpoint rule per ray (R8).
 *   Normalization box (R11): x -> (x - rot_center_x)/r, y -> y/r,
 *   z -> (z - (z_lo+z_hi)/2)/((z_hi-z_lo)/2), t -> (t - (t_lo+t_hi)/2)/((t_hi-t_lo)/2);
 *   a zero-width range maps that coordinate to 0.  NaN z_lo / z_hi: derived from the geometry —
 *   the detector z extent [-C_z, -C_z + n_rows dz], scaled for cone beam by (sod + r)/(sod + odd)
 *   (the far side of the FOV cylinder); NaN t_lo / t_hi: the first / last view time.
 * Invariants: sod > 0, odd >= 0, pixel pitches > 0, fov_radius > 0,
 *   fov_radius < sod, sub_x, sub_z >= 1, samples_per_ray >= 1 (a multiple of 32 on the BF16 path,
 *   checked by whichever of set_geometry / set_field_weights comes second),
 *   n_rows, n_cols >= 1, z_hi >= z_lo, t_hi >= t_lo. */
typedef struct {
  int32_t beam;            /* dinr_beam */
  int32_t n_rows, n_cols;
  int32_t sub_x, sub_z;
  int32_t samples_per_ray;
  double sod, odd;
  double pixel_dx, pixel_dz;
  double offset_cx, offset_cz;
  double fov_radius, rot_center_x;
  double z_lo, z_hi;
  double t_lo, t_hi;
} dinr_geometry;

/* DINR field network: GRFF with n_freq = C frequencies (width H = 2C), L =
 * n_layers FC(H->H)+Swish layers, FC head H->1 times mu0 (applied once, R6).
 * Supported on the BF16 path: H in {64, 128, 256}, 1 <= L <= 64 (L <= 27 at H = 256, where every
 * layer's bias sits in the tensor-core kernels' shared memory; DINR_EINVAL beyond); FP32_VERIFY: any
 * even H <= 256.
 * Accuracy envelope of the BF16 path (bf16 tensor-core operands, fp32 accumulation and epilogue):
 * against the fp64 oracle, projections within 2e-3 and gradients within 1e-2 (relative L-inf per
 * parameter tensor, R23) for L <= 3 at H = 64, L <= 4 at H = 128 and L <= 6 at H = 256
 * (the BASELINE depths), on inputs whose sums do not cancel (R23b: a bias gradient is a plain sum of
 * deltas; residuals of both signs that nearly cancel amplify any bf16 error by sum|d| / |sum d|).
 * Deeper networks run with the error growing with depth (measured 1.5e-2 gradients at H = 64, L = 6).
 * FP32_VERIFY: projections within 1e-5, gradients within 1e-4.
 * mu0 > 0.  combine: dinr_combine.  precision: dinr_precision. */
typedef struct {
  int32_t n_freq;
  int32_t n_layers;
  int32_t width;           /* must equal 2*n_freq */
  int32_t combine;
  int32_t precision;
  int32_t reserved;        /* 0 */
  double mu0;
} dinr_field_desc;

/* Trainable parameter count P = L(H^2+H)+H+1.  Layout of the flat fp32
 * parameter / gradient vector (D5): for l = 1..L: W_l (H x H row-major [out][in]), b_l (H);
 * then w_o (H), b_o (1). */
int64_t dinr_param_count(int32_t n_freq, int32_t n_layers);

/* Create a context on CUDA device `device` (must be compute capability 10.0). */
dinr_status dinr_create(int device, dinr_ctx **out);
dinr_status dinr_destroy(dinr_ctx *ctx);
/* Text of the last error on this context (valid until the next call on it). */
const char *dinr_last_error(const dinr_ctx *ctx);
const char *dinr_status_string(dinr_status s);

/* Geometry and view schedule: theta_rad[M] (view angles; source and detector rotate
 * anticlockwise by theta_k about (x_s0, 0), eq:rotxsk-rotydk P:88-106, R4) and t[M]
 * (acquisition times, t_i = T_m for every pixel of view m, non-decreasing).
 * Host arrays, copied before return (synchronous).  cos/sin of theta are taken on the host. */
dinr_status dinr_set_geometry(dinr_ctx *ctx, const dinr_geometry *g, const double *theta_rad,
                              const double *t, int64_t M);

/* Sample placement for the following calls (host state, no device work; default MIDPOINT).
 * JITTER draws every uniform from Philox4x32-10 with key = seed (lo, hi words) and counter
 * (w0, R lo, R hi, step) for global ray R = pixel index * S + s: w0 = j for sample j's offset
 * u_j = (x >> 8) 2^-24 of output word x; w0 = 0xFFFFFFFF for the sub-pixel offsets (ux, uz)
 * from output words x, y.  Results depend only on (seed, step, pixel index), not on the batch.
 * Error: DINR_EINVAL for an unknown mode. */
dinr_status dinr_set_sampling(dinr_ctx *ctx, dinr_sampling mode, uint64_t seed, uint32_t step);

/* ---------------------------------------------------------------------------------------------
 * N4 inference voxelization: the trained field on a regular 3D grid at
 * a view time.  Voxel (i, j, k), 0 <= i < nx etc., has centre
 *   (x0 + (i + 1/2) vx, y0 + (j + 1/2) vy, z0 + (k + 1/2) vz)    (object frame, lengths as geometry). */
typedef struct {
  int64_t nx, ny, nz;
  double x0, y0, z0;  /* lower corner of voxel (0, 0, 0) */
  double vx, vy, vz;  /* voxel size */
} dinr_voxel_grid;

/* The paper's grid: voxel = detector pixel / geometric magnification (1 for
 * parallel, (sod + odd) / sod for fan and cone: source-to-detector over source-to-object), i.e.
 * vx = vy = pixel_dx / mag, vz = pixel_dz / mag, covering the FOV box [x_s0 - r, x_s0 + r] x
 * [-r, r] x [z_lo, z_hi] with nx = ny = ceil(2r / vx), nz = ceil((z_hi - z_lo) / vz), centred on
 * the box.  Host only; requires dinr_set_geometry (else DINR_ESTATE). */
dinr_status dinr_default_grid(dinr_ctx *ctx, dinr_voxel_grid *out);

/* mu(x, t) = mu0 (w_o . h_L + b_o) (R6) at the voxel centres of the z planes
 * [k_begin, k_begin + k_count) at time t (normalized like the training samples):
 *   out_dev[((k - k_begin) ny + j) nx + i]  fp32, device memory of nx ny k_count floats;
 * 0 for centres outside the FOV cylinder (x - x_s0)^2 + y^2 <= r^2 (R25).  Precision as set by
 * dinr_set_field_weights.  Stream-ordered.  DINR_EINVAL for an empty / out-of-range slab. */
dinr_status dinr_voxelize(dinr_ctx *ctx, const dinr_voxel_grid *grid, double t, int64_t k_begin, int64_t k_count,
                          float *out_dev, void *stream);

/* Volumes at the view times t_m, m in [view_begin, view_begin + n_views) (the paper voxelizes at
 * the acquisition times), streamed to a raw little-endian fp32 file laid out [m][k][j][i]:
 * slabs of slab_planes z planes are computed on the GPU while the previous slab is copied to
 * pinned host memory and written (double buffering).  Synchronous; DINR_EINVAL on a bad range,
 * DINR_ECUDA on an I/O error (message names the file). */
dinr_status dinr_voxelize_to_file(dinr_ctx *ctx, const dinr_voxel_grid *grid, int64_t view_begin, int64_t n_views,
                                  const char *path, int64_t slab_planes);

/* Field weights: B_dev = GRFF matrix (C x 4 fp32, columns t,z,y,x, frozen, R12);
 * params_dev = P fp32 trainable parameters (D5 layout).  Packs bf16 tensor-core operands on
 * `stream` (stream-ordered; the caller may overwrite params_dev after this on the same
 * stream).  Requires dinr_set_geometry first (else DINR_ESTATE). */
dinr_status dinr_set_field_weights(dinr_ctx *ctx, const dinr_field_desc *f, const float *B_dev,
                                   const float *params_dev, void *stream);

/* Forward projection of n flat pixel indices i = m*N + n (N = n_rows*n_cols):
 *   fhat_dev[n]  log-domain projection -log(I/I0) (eq:logbeerslaw; BEER or LINEAR combine);
 *   p_sub_dev    [n*S] per-sub-ray line integrals p_s = (chord_s/N_s) sum_j M(r_j) (eq:estforwmod
 *                with R7), or NULL;
 *   I0_dev/Ihat_dev: optional [n] blank intensities and predicted intensities
 *                Ihat = I0 exp(-fhat) (eq:beerstransavg), both NULL or both set.
 * n = 0 is legal (no work).  idx_dev is int64. */
dinr_status dinr_project(dinr_ctx *ctx, const int64_t *idx_dev, int64_t n, float *fhat_dev,
                         float *p_sub_dev, const float *I0_dev, float *Ihat_dev, void *stream);

/* Local loss and gradient (eq:mainsqdist, eq:localoptfunc P:3261-3297; eq:partiald
 * P:406-423): L = (1/n) sum_i (y_i - fhat_i)^2 over the n pixels; grad_dev[0..P-1] =
 * dL/dgamma (D5 layout), grad_dev[P] = L.  accumulate = 0 overwrites, 1 adds.  n = 0 writes
 * zeros (every rank must still join dinr_allreduce_grads). */
dinr_status dinr_project_and_grad(dinr_ctx *ctx, const int64_t *idx_dev, int64_t n,
                                  const float *y_dev, float *grad_dev, int accumulate,
                                  void *stream);

/* Same as dinr_project_and_grad but with HOST buffers (end-to-end entry point): copies
 * idx_host[n] and y_host[n] to the device, runs the step on `stream`, optionally averages
 * the gradient over the communicator (allreduce != 0), and copies grad (P+1 floats) back to
 * grad_host.  Synchronizes `stream` before returning.  Pinned host memory is fastest. */
dinr_status dinr_project_and_grad_host(dinr_ctx *ctx, const int64_t *idx_host, int64_t n,
                                       const float *y_host, float *grad_host, int allreduce,
                                       void *stream);

/* Optimizer step (NEXT row N1; "We use the Adam optimizer"):
 * one fused kernel updates params_dev in place with Adam (bias-corrected, step >= 1),
 *   m <- b1 m + (1-b1) g, v <- b2 v + (1-b2) g^2, p <- p - lr mhat/(sqrt(vhat)+eps),
 * and re-packs the context's bf16 tensor-core weight images from the new values (so it
 * replaces dinr_set_field_weights after the first call).  params_dev, m_dev, v_dev: P fp32
 * each (D5 layout, caller-owned); grad_dev: at least P fp32 (slot P, the loss, is ignored).
 * Requires dinr_set_field_weights first (DINR_ESTATE); count must equal P (DINR_EINVAL). */
dinr_status dinr_adam_step(dinr_ctx *ctx, float *params_dev, const float *grad_dev, float *m_dev, float *v_dev,
                           int64_t count, double lr, double beta1, double beta2, double eps, int64_t step,
                           void *stream);

/* ---- N1 epoch loop (lr schedule P:540-542; reading R27 in DESIGN.md) ----------
 * Each process k draws |Omega_k| = batch pixels per iteration (eq:localoptfunc, eq:totbatch:
 * Omega* = world * batch), without replacement through a per-epoch pseudo-random permutation
 * (SPEC S:389), computes the local mean loss and gradient, the gradients are averaged
 * over the processes (dinr_allreduce_grads), and every process applies the same Adam step with
 * lr = lr0 * lr_decay^epoch.  One epoch = ceil(M N / Omega*) iterations; the last
 * iteration of an epoch wraps to the start of the same permutation so that every process always
 * takes exactly `batch` pixels (equal |Omega_k|).
 * sharding DINR_SHARD_VIEWS: process `rank` owns views rank, rank + world, ... and
 *   permutes the nv N positions of its shard (nv = ceil((M - rank) / world)); its y source is that
 *   shard, nv N floats stored view by view.
 * sharding DINR_SHARD_GLOBAL: one permutation of all M N pixels, each iteration's Omega* positions
 *   split contiguously over the processes; the y source is all M N floats.
 * The permutation: an 8-round Feistel network over Philox4x32-10 with cycle walking (k_sampler.cuh;
 * the oracle implements the same generator independently). */
typedef enum { DINR_SHARD_VIEWS = 0, DINR_SHARD_GLOBAL = 1 } dinr_sharding;

typedef struct {
  uint64_t seed;    /* permutation key */
  int32_t rank;     /* this process (0 <= rank < world) */
  int32_t world;    /* number of processes K; > 1 requires dinr_comm_init with the same world */
  int32_t sharding; /* dinr_sharding */
  int32_t reserved; /* 0 */
  int64_t batch;    /* |Omega_k| >= 1 */
  double lr0;       /* initial learning rate (paper: 0.001) */
  double lr_decay;  /* per-epoch factor (paper: 0.95) */
  double beta1, beta2, eps; /* Adam (0.9, 0.999, 1e-8) */
} dinr_train_desc;

/* ceil(M N / (world * batch)).  DINR_ESTATE before dinr_set_geometry; DINR_EINVAL for a bad desc. */
dinr_status dinr_iterations_per_epoch(dinr_ctx *ctx, const dinr_train_desc *desc, int64_t *out);

/* The batch of iteration `iteration` of epoch `epoch` for desc->rank: idx_dev[batch] pixel
 * indices and, when y_src_dev is not null, y_dev[batch] = the measured values gathered from the
 * y source described above.  Stream-ordered, one kernel.  DINR_EINVAL for negative epoch /
 * iteration, a bad desc or null outputs. */
dinr_status dinr_sample_batch(dinr_ctx *ctx, const dinr_train_desc *desc, int64_t epoch, int64_t iteration,
                              const float *y_src_dev, int64_t *idx_dev, float *y_dev, void *stream);

/* Runs global iterations first .. first + count - 1 (iteration g is iteration g mod I of epoch
 * g / I, I = dinr_iterations_per_epoch; Adam step g + 1): sample, dinr_project_and_grad,
 * dinr_allreduce_grads when world > 1, dinr_adam_step with the epoch's lr.  params_dev, m_dev,
 * v_dev: P fp32 (caller-owned, updated in place; the context's weight images follow them);
 * grad_dev: P + 1 fp32 scratch (holds the last averaged gradient and loss on return);
 * loss_dev: count fp32, the global mean loss of each iteration (eq:localoptfunc averaged over
 * the processes).  All stream-ordered on `stream`, no host synchronization.  Requires
 * dinr_set_field_weights (DINR_ESTATE), and dinr_comm_init with desc->world processes when
 * world > 1 (DINR_ESTATE). */
dinr_status dinr_train_iterations(dinr_ctx *ctx, const dinr_train_desc *desc, int64_t first, int64_t count,
                                  const float *y_src_dev, float *params_dev, float *m_dev, float *v_dev,
                                  float *grad_dev, float *loss_dev, void *stream);

/* Analytic phantom primitive (NEXT row N2): kind 0 = indicator ellipsoid (value mu), 1 = smooth
 * ellipsoid mu_c (1 - rho^2)^2, 2 = Gaussian A exp(-rho^2/2) with sigmas = axes.  Axis-aligned in
 * the object frame, centre(t) = center + velocity t, axes(t) = axes + axes_rate t. */
typedef struct {
  int32_t kind;
  int32_t reserved;
  double value;
  double center[3], velocity[3], axes[3], axes_rate[3];
} dinr_primitive;

/* Measured-data synthesis (N2): exact line integrals of the phantom along every sub-ray of the
 * n pixels (fp64, closed forms, on the K1 ray records), combined per pixel with `combine`
 * (dinr_combine) into fhat_dev[n] = -log(I/I0); p_sub_dev[n*S] (or NULL) gets the noiseless
 * sub-ray integrals.  noise_frac > 0 adds transmission-space Gaussian noise of std
 * noise_frac*sqrt(T) (eq:forwmod P:261-272, R24) from a counter-based generator keyed by
 * (seed, pixel index) -- reproducible and independent of launch order.  prims_host: host array
 * of n_prims (<= 64) primitives, copied before return.  Requires dinr_set_geometry. */
dinr_status dinr_phantom_project(dinr_ctx *ctx, const dinr_primitive *prims_host, int32_t n_prims,
                                 const int64_t *idx_dev, int64_t n, int32_t combine, double noise_frac,
                                 uint64_t seed, float *fhat_dev, float *p_sub_dev, void *stream);

/* fp64 ray records of kernel K1 (geometry / ray setup) for n pixels: rec_dev[n*S*9] =
 * {o.x,o.y,o.z, d.x,d.y,d.z, delta_min, delta_max, chord} per sub-ray, where o is the
 * rotated source, d = rotated detector point - o, [delta_min, delta_max] the FOV bounds
 * clamped to [0,1] (eq:solvquaddelta/eq:deltaminmax; miss -> (0,0)) and chord
 * = |det - src|_2 (delta_max - delta_min) (eq:arclength read as the Euclidean norm, R1). */
dinr_status dinr_ray_records(dinr_ctx *ctx, const int64_t *idx_dev, int64_t n, double *rec_dev,
                             void *stream);

/* Data-parallel gradient averaging: 128-byte NCCL unique id (rank 0 creates
 * it, the caller broadcasts it), communicator init, and an in-place
 * ncclAllReduce(ncclFloat32, ncclAvg) of count floats on `stream` (gradients and the loss
 * slot are averaged in the same call, R16). */
dinr_status dinr_nccl_unique_id(void *out_128_bytes);
dinr_status dinr_comm_init(dinr_ctx *ctx, const void *unique_id_128_bytes, int rank, int world);
dinr_status dinr_allreduce_grads(dinr_ctx *ctx, float *grad_dev, int64_t count, void *stream);

/* Synchronizes the device and reports sticky device-side errors (DINR_ERANGE), then clears. */
dinr_status dinr_get_device_status(dinr_ctx *ctx);

/* Instrumentation.  dinr_set_timing(ctx, 1) brackets every kernel this library launches
 * with CUDA events on the launching stream; dinr_read_timing() synchronizes and returns, for
 * kernel class `which` (0 = ray setup, 1 = forward MLP, 2 = loss, 3 = backward MLP,
 * 4 = dW GEMM, 5 = gradient assembly, 6 = weight pack, 7 = all-reduce), the summed device
 * milliseconds and the launch count since the last reset (reset != 0 clears after reading).
 * dinr_launch_count() returns the number of kernels launched by this context so far. */
dinr_status dinr_set_timing(dinr_ctx *ctx, int enable);
dinr_status dinr_read_timing(dinr_ctx *ctx, int which, double *ms, int64_t *launches, int reset);
int64_t dinr_launch_count(const dinr_ctx *ctx);

/* Which training path dinr_project_and_grad takes for a batch of n pixels with the current
 * geometry and weights (host query, no device work): *fused_kernel = 0 split path (K2/K3/K5),
 * 1 one-stream fused kernel, 2 two-stream fused kernel; *fused_dw_layers = number of top layers
 * whose dW accumulate inside the fused kernel (the rest go through the dW GEMM).  For the
 * roofline bookkeeping of bench.py.  DINR_ESTATE before weights are set. */
dinr_status dinr_train_path(dinr_ctx *ctx, int64_t n, int32_t *fused_kernel, int32_t *fused_dw_layers);

/* Algorithmic work of the training step per kernel class, for the roofline (only
 * what the method must compute -- L forward, L - 1 dX and L dW H x H GEMMs per sample, i.e.
 * 2 (3L - 1) H^2 FLOP; recomputed GEMMs and padding are not counted).  gemm_layers[which]
 * (which = the dinr_read_timing classes 0..7) receives the number of those H x H GEMMs per
 * sample that the kernels of that class perform for a batch of n pixels on the current path;
 * the entries sum to 3L - 1.  Host query, no device work.  DINR_ESTATE before weights are set;
 * DINR_EINVAL for a null array or n < 0. */
dinr_status dinr_train_gemm_layers(dinr_ctx *ctx, int64_t n, int32_t gemm_layers[8]);

#ifdef __cplusplus
}
#endif
#endif /* DINR_H */
