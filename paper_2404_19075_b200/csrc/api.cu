// api.cu -- libdinr.so: the C ABI of include/dinr.h.  Host-side validation, scratch
// management, kernel launches (all stream-ordered on the caller's stream), NCCL plumbing and
// instrumentation.  Kernels live in the included .cuh files (single translation unit).
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "internal.cuh"
#include "k_geometry.cuh"
#include "k_simt.cuh"
#include "k_small.cuh"
#include "k_tc_dw.cuh"
#include "k_tc_dwz.cuh"
#include "k_tc_mlp.cuh"
#include "k_fused.cuh"
#include "k_fused2.cuh"
#include "k_dw01.cuh"
#include "k_tc_fwd2.cuh"
#include "k_tc_bwd2.cuh"
#include "k_tc_fwd3.cuh"
#include "k_tc_bwd3.cuh"
#include "k_infer.cuh"
#include "k_phantom.cuh"
#include "k_sampler.cuh"
#include "nccl_dl.cuh"

using namespace dinr;

namespace {

thread_local std::string g_static_err;

dinr_status fail(dinr_ctx *c, dinr_status s, const std::string &msg) {
  if (c) c->err = msg;
  return s;
}

#define CUDA_TRY(c, expr)                                                                     \
  do {                                                                                        \
    cudaError_t _e = (expr);                                                                  \
    if (_e != cudaSuccess) return fail((c), DINR_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

// Kernel-launch bracket: counts the launch and, when timing is on, records CUDA events on
// the launching stream around it.
struct Launch {
  dinr_ctx *c;
  int cls;
  cudaStream_t st;
  cudaEvent_t a = nullptr, b = nullptr;
  Launch(dinr_ctx *c_, int cls_, cudaStream_t st_) : c(c_), cls(cls_), st(st_) {
    if (cls != T_AR) c->launches++;  // NCCL's kernel is not ours
    if (c->timing) {
      a = take();
      b = take();
      cudaEventRecord(a, st);
    }
  }
  cudaEvent_t take() {
    if (c->event_pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = c->event_pool.back();
    c->event_pool.pop_back();
    return e;
  }
  ~Launch() {
    if (a) {
      cudaEventRecord(b, st);
      c->pending.push_back({cls, a, b});
    }
  }
};

bool is_fin(double x) { return std::isfinite(x); }

// Carve a scratch arena into 256-B aligned pieces.  With DINR_GUARDS set (a debugging mode: the
// pool has no compute-sanitizer), every piece is preceded by a 4 KB guard band that ensure_plan fills
// with 0xA5 and dinr_get_device_status checks: any write past the end of a scratch buffer lands in a
// band and is reported as DINR_EDEVICE.
constexpr size_t kGuardBytes = 4096;
bool guards_on() {
  static const bool on = std::getenv("DINR_GUARDS") != nullptr;
  return on;
}
struct Arena {
  uint8_t *base;
  size_t off = 0;
  std::vector<size_t> *bands = nullptr;  // guard band offsets (DINR_GUARDS)
  explicit Arena(void *b) : base((uint8_t *)b) {}
  template <class T>
  T *take(size_t count) {
    off = (off + 255) & ~size_t(255);
    if (guards_on()) {
      if (bands) bands->push_back(off);
      off += kGuardBytes;
    }
    T *p = base ? reinterpret_cast<T *>(base + off) : nullptr;
    off += count * sizeof(T);
    return p;
  }
};

struct Plan {
  int64_t n, n_rays, nsamp, n_tiles;
  int nc;
  int grid_tc;
  int ksplit, nmb;
  int ks0, ks1;  // dW GEMM K-splits of layer 0 / the other layers (see launch_tc_dw)
  int ksplit_simt;
  int nloss;
  // fused training path (k_fused): nf top layers' dW in TMEM, nu = L - nf through K5
  bool fused, fused2;  // fused2: two concurrent tile streams (k_fused2)
  bool dw01;           // layers 0 and 1 unfused, both inputs recomputed by k_dw01 (no input stash)
  bool feat0;          // the dW GEMM recomputes layer 0's input (needs N_s a power of two)
  bool zall;           // H = 256 split path: y = z/2 stash only; K3 / the dW GEMM recompute swish', h
  int nf, nu, grid_f, dw_layers;
  uint8_t *ring;
  float *dwf, *dbf;
  // carved pointers
  float4 *rec32;
  uint2 *rid;   // global ray ids (N3 keys)
  Jitter jit;   // N3 sample placement handed to the MLP kernels
  float *pchunk, *u, *fhat, *loss_part, *head_part, *dw_part, *db_part, *colsum;
  float *smu;  // fp32 verify with N_s % 32 != 0: per-sample mu before the per-ray sums
  float *db3;  // zall: K3's per-CTA bias-gradient partials [L][2][grid_tc][128]
  float *wq;  // per-ray quadrature weight (K1 -> K4)
  uint8_t *hstash, *dstash, *zstash;
  float *sh, *sz, *sd;
  int64_t *idx_dev;
  float *y_dev, *grad_dev;
};

constexpr size_t kMaxSmem = 227 * 1024;  // dynamic shared memory per CTA (sm_100)

bool fused2_fits(const dinr_ctx *c) {
  const size_t smem = c->H == 64 ? Fused2Layout<64>::smem_bytes(c->L) : Fused2Layout<128>::smem_bytes(c->L);
  return smem <= kMaxSmem;
}

bool fused1_fits(const dinr_ctx *c) {
  const size_t smem = c->H == 64 ? FusedLayout<64>::smem_bytes(c->L) : FusedLayout<128>::smem_bytes(c->L);
  return smem <= kMaxSmem;
}

bool use_fused(const dinr_ctx *c) {
  static const bool off = std::getenv("DINR_NO_FUSED") != nullptr;
  const int ns = c->geom.samples_per_ray, sn = c->S * ns;
  // the fused kernels keep W_1..W_{L-1} resident: deep networks that fit neither take the split path
  return !off && c->field.precision == DINR_BF16 && c->H <= 128 && sn <= 256 && 256 % sn == 0 && (ns & (ns - 1)) == 0 &&
         (fused2_fits(c) || fused1_fits(c));
}

bool use_fused2(const dinr_ctx *c) {
  static const bool off = std::getenv("DINR_FUSED_V1") != nullptr;
  return fused2_fits(c) && !(off && fused1_fits(c));
}

// the H = 256 split path's K2 on CTA pairs (k_tc_fwd3), with the y-only stash (zall)
bool fwd3_on() {
  static const bool off = std::getenv("DINR_NO_FWD3") != nullptr || std::getenv("DINR_NO_FWD2") != nullptr;
  return !off;
}

int loss_blocks_for(int64_t n) { return (int)std::max<int64_t>(1, (n + kLossThreads - 1) / kLossThreads); }

int tc_occupancy(const dinr_ctx *c) {
  // one CTA per SM for H >= 128 (shared memory); up to 4 for H = 64
  return c->H == 64 ? 4 : 1;
}

bool tc_resident(int H, int L) { return (size_t)L * H * H * 2 + (size_t)H * 256 <= 180 * 1024; }

size_t plan_layout(dinr_ctx *c, int64_t n, bool train, bool host_io, Plan &pl, void *base,
                   std::vector<size_t> *bands = nullptr) {
  Arena ar(base);
  ar.bands = bands;
  pl.n = n;
  pl.n_rays = n * c->S;
  pl.nsamp = pl.n_rays * c->geom.samples_per_ray;
  // ray-sum partials per ray: 32-sample chunks, or (fp32 verify with N_s not a multiple of 32) one per ray
  const bool whole_warps = c->geom.samples_per_ray % kChunk == 0;
  pl.nc = whole_warps ? c->geom.samples_per_ray / kChunk : 1;
  pl.n_tiles = (pl.nsamp + 127) / 128;
  pl.grid_tc = (int)std::max<int64_t>(1, std::min<int64_t>(pl.n_tiles, (int64_t)c->sm_count * tc_occupancy(c)));
  pl.nmb = c->H == 256 ? 2 : 1;
  // dW GEMM K-split: one wave of nmb * L * ksplit <= sm_count CTAs (one CTA per SM; a second
  // partial wave would double the kernel time)
  pl.ksplit = (int)std::max<int64_t>(1, std::min<int64_t>(pl.n_tiles, c->sm_count / (pl.nmb * c->L)));
  pl.ks0 = pl.ks1 = pl.ksplit;
  pl.ksplit_simt = (int)std::max<int64_t>(1, std::min<int64_t>(64, pl.nsamp / 1024));
  pl.nloss = loss_blocks_for(n);
  const int H = c->H, L = c->L;
  pl.rec32 = ar.take<float4>(2 * pl.n_rays + 2);
  pl.rid = ar.take<uint2>(pl.n_rays + 1);
  pl.jit.rid = c->sampling == DINR_JITTER ? pl.rid : nullptr;
  pl.jit.seed_lo = (uint32_t)c->seed;
  pl.jit.seed_hi = (uint32_t)(c->seed >> 32);
  pl.jit.step = c->step;
  pl.pchunk = ar.take<float>(whole_warps ? pl.nsamp / kChunk + 1 : pl.n_rays + 1);
  pl.smu = whole_warps ? nullptr : ar.take<float>(pl.nsamp + 1);
  pl.u = ar.take<float>(pl.n_rays + 1);
  pl.wq = ar.take<float>(pl.n_rays + 1);
  pl.fhat = ar.take<float>(n + 1);
  pl.loss_part = ar.take<float>(pl.nloss + 1);
  const bool simt = c->field.precision == DINR_FP32_VERIFY;
  // H = 256 split path with k_tc_fwd3 (y-only stash): the dW GEMM k_tc_dwz runs one CTA per
  // (layer, K-split) for both output blocks
  // (experiment, off by default: measured no faster -- the forward saves its writes but K3 and the
  // dW GEMM redo the MUFU work)
  static const bool zall_on = std::getenv("DINR_ZALL") != nullptr;
  const bool zall_path = train && !simt && !use_fused(c) && c->H == 256 && fwd3_on() && zall_on &&
                         Fwd3Layout::smem_bytes(c->L) <= kMaxSmem;
  if (zall_path) pl.ks0 = pl.ks1 = pl.ksplit = (int)std::max<int64_t>(1, std::min<int64_t>(pl.n_tiles, c->sm_count / c->L));
  static const bool split_feat0 = std::getenv("DINR_SPLIT_FEAT0") != nullptr;
  const bool sfeat0 = split_feat0 && !zall_path && train && !simt && !use_fused(c) && c->L >= 2;
  if (sfeat0) {  // layer-0 CTAs rebuild the features (MUFU): give them w0 x the K-split of the others
    static const double w0 = std::getenv("DINR_DW_W0") ? std::atof(std::getenv("DINR_DW_W0")) : 2.0;
    const int sm = c->sm_count / pl.nmb;
    pl.ks0 = std::max(1, (int)(sm * w0 / (w0 + c->L - 1) + 0.5));
    pl.ks1 = std::max(1, (sm - pl.ks0) / (c->L - 1));
    pl.ks0 = (int)std::min<int64_t>(pl.ks0, pl.n_tiles);
    pl.ks1 = (int)std::min<int64_t>(pl.ks1, pl.n_tiles);
    pl.ksplit = std::max(pl.ks0, pl.ks1);
  }
  const int ks = simt ? pl.ksplit_simt : pl.ksplit;
  pl.head_part = ar.take<float>((size_t)std::max(pl.grid_tc, ks) * (H + 1));
  pl.dw_part = pl.db_part = nullptr;
  pl.hstash = pl.dstash = pl.zstash = nullptr;
  pl.sh = pl.sz = pl.sd = pl.colsum = nullptr;
  if (train) {
    pl.dw_part = ar.take<float>((size_t)L * pl.nmb * ks * 128 * H);
    pl.db_part = ar.take<float>((size_t)L * pl.nmb * ks * 128);
  }
  pl.fused = train && use_fused(c);
  pl.fused2 = pl.fused && use_fused2(c);
  pl.dw01 = false;
  // layer 0's features recomputed by the dW GEMM instead of stashed: on the fused path (for the
  // split path, H = 256, the recompute of 128 frequencies costs more than the stash traffic)
  pl.feat0 = pl.fused;
  pl.zall = false;
  pl.db3 = nullptr;
  pl.nf = pl.nu = pl.grid_f = 0;
  pl.dw_layers = L;
  pl.ring = nullptr;
  pl.dwf = pl.dbf = nullptr;
  if (pl.fused) {
    // the fused kernels work in pixel groups of two 128-sample tiles: the stash (and the dW
    // kernels over it) cover whole groups; the tile past an odd tile count holds only invalid
    // samples, whose delta is exactly zero, so it adds nothing to dW / db
    pl.n_tiles = 2 * ((pl.nsamp + 255) / 256);
    pl.nf = std::min(std::min(L, 4), 512 / H - (pl.fused2 ? 2 : 1));  // <= 4: per-thread db registers
    pl.nu = L - pl.nf;
    pl.dw_layers = pl.nu;
    const int64_t n_groups = (pl.nsamp + 255) / 256;
    pl.grid_f = (int)std::max<int64_t>(1, std::min<int64_t>(n_groups, c->sm_count));
    // dW GEMM grid: layer 0 recomputes its input (GRFF features) and gets w0 x the CTAs of a
    // layer that streams both operands from HBM
    static const bool no_dw01 = std::getenv("DINR_NO_DW01") != nullptr;
    pl.dw01 = pl.fused2 && pl.nu == 2 && H == 128 && !no_dw01;
    if (pl.dw01) {
      pl.ks0 = pl.ks1 = pl.ksplit = (int)std::min<int64_t>(c->sm_count, pl.n_tiles);
    } else if (pl.nu > 0) {
      static const double w0 = std::getenv("DINR_DW_W0") ? std::atof(std::getenv("DINR_DW_W0")) : 2.0;
      const int sm = c->sm_count;
      pl.ks0 = pl.nu == 1 ? sm : std::max(1, (int)(sm * w0 / (w0 + pl.nu - 1) + 0.5));
      pl.ks1 = pl.nu == 1 ? 1 : std::max(1, (sm - pl.ks0) / (pl.nu - 1));
      pl.ks0 = (int)std::min<int64_t>(pl.ks0, pl.n_tiles);
      pl.ks1 = (int)std::min<int64_t>(pl.ks1, pl.n_tiles);
      pl.ksplit = std::max(pl.ks0, pl.nu > 1 ? pl.ks1 : 1);
    } else {
      pl.ksplit = 1;
    }
    pl.ring = ar.take<uint8_t>((size_t)pl.grid_f * 2 * (L + pl.nf) * H * 256);
    pl.dwf = ar.take<float>((size_t)pl.nf * pl.grid_f * 128 * H);
    pl.dbf = ar.take<float>((size_t)pl.nf * pl.grid_f * 128);
    pl.head_part = ar.take<float>((size_t)pl.grid_f * (H + 1));
    pl.loss_part = ar.take<float>((size_t)pl.grid_f + 1);
    if (pl.nu > 0) {
      pl.hstash = ar.take<uint8_t>((size_t)pl.nu * pl.n_tiles * H * 256);
      pl.dstash = ar.take<uint8_t>((size_t)pl.nu * pl.n_tiles * H * 256);
      pl.dw_part = ar.take<float>((size_t)pl.nu * pl.ksplit * 128 * H);
      pl.db_part = ar.take<float>((size_t)pl.nu * pl.ksplit * 128);
    }
  } else if (!simt && train) {
    // the split path's training forward runs tiles in pairs (k_tc_fwd2): an even tile count; the
    // padding tile holds only invalid samples, whose upstream factor and so delta are exactly zero
    // (k_tc_fwd3, H = 256, works in CTA pairs on 4 tiles at a time: a multiple of 4)
    pl.n_tiles = H == 256 ? 4 * ((pl.nsamp + 511) / 512) : 2 * ((pl.nsamp + 255) / 256);
    // H = 256 with k_tc_fwd3: the forward stashes y = z / 2 of every layer (fp16) and nothing else
    pl.zall = zall_path;
    // layer 0's dW operand (the GRFF features) recomputed by the dW GEMM instead of stashed by K2
    pl.feat0 = pl.zall || sfeat0;
    if (!pl.zall) pl.hstash = ar.take<uint8_t>((size_t)L * pl.n_tiles * H * 256);
    if (pl.zall) pl.db3 = ar.take<float>((size_t)L * 2 * pl.grid_tc * 128);
    pl.dstash = ar.take<uint8_t>((size_t)L * pl.n_tiles * H * 256);
    pl.zstash = ar.take<uint8_t>((size_t)L * pl.n_tiles * H * 256);
  }
  if (simt) {
    pl.sh = ar.take<float>((size_t)(L + 1) * pl.nsamp * H);
    pl.sz = ar.take<float>((size_t)L * pl.nsamp * H);
    pl.sd = ar.take<float>((size_t)pl.nsamp * H);
  }
  pl.idx_dev = nullptr;
  pl.y_dev = pl.grad_dev = nullptr;
  if (host_io) {
    pl.idx_dev = ar.take<int64_t>(n + 1);
    pl.y_dev = ar.take<float>(n + 1);
    pl.grad_dev = ar.take<float>(c->P + 1);
  }
  return ar.off + 1024;
}

dinr_status ensure_plan(dinr_ctx *c, int64_t n, bool train, bool host_io, Plan &pl) {
  size_t need = plan_layout(c, n, train, host_io, pl, nullptr);
  if (need > c->scratch_cap) {
    if (c->scratch) cudaFree(c->scratch);
    c->scratch = nullptr;
    c->scratch_cap = 0;
    size_t cap = need + need / 4;
    if (cudaMalloc(&c->scratch, cap) != cudaSuccess) {
      cudaGetLastError();
      return fail(c, DINR_ENOMEM, "scratch allocation of " + std::to_string(cap) + " bytes failed");
    }
    c->scratch_cap = cap;
  }
  if (guards_on()) {
    std::vector<size_t> bands;
    plan_layout(c, n, train, host_io, pl, c->scratch, &bands);
    bands.push_back((need - 1024 + 255) & ~size_t(255));  // tail band: after the last buffer (inside the slack)
    c->guard_bands = bands;
    for (size_t b : bands)
      if (b + kGuardBytes <= c->scratch_cap) CUDA_TRY(c, cudaMemset((uint8_t *)c->scratch + b, 0xA5, kGuardBytes));
    return DINR_OK;
  }
  plan_layout(c, n, train, host_io, pl, c->scratch);
  return DINR_OK;
}

// DINR_GUARDS: every guard band still holds 0xA5 (checked by dinr_get_device_status)
bool guards_intact(dinr_ctx *c, size_t *bad) {
  std::vector<uint8_t> h(kGuardBytes);
  for (size_t b : c->guard_bands) {
    if (b + kGuardBytes > c->scratch_cap) continue;
    if (cudaMemcpy(h.data(), (uint8_t *)c->scratch + b, kGuardBytes, cudaMemcpyDeviceToHost) != cudaSuccess) return false;
    for (size_t i = 0; i < kGuardBytes; ++i)
      if (h[i] != 0xA5) {
        *bad = b + i;
        return false;
      }
  }
  return true;
}

GeomParams geom_params(const dinr_ctx *c) {
  const dinr_geometry &g = c->geom;
  GeomParams gp;
  gp.beam = g.beam;
  gp.n_rows = g.n_rows;
  gp.n_cols = g.n_cols;
  gp.sub_x = g.sub_x;
  gp.sub_z = g.sub_z;
  gp.n_s = g.samples_per_ray;
  gp.sod = g.sod;
  gp.odd = g.odd;
  gp.dx = g.pixel_dx;
  gp.dz = g.pixel_dz;
  gp.cx = g.offset_cx;
  gp.cz = g.offset_cz;
  gp.r = g.fov_radius;
  gp.xs0 = g.rot_center_x;
  gp.zc = 0.5 * (g.z_lo + g.z_hi);
  gp.zh = 0.5 * (g.z_hi - g.z_lo);
  gp.tc = 0.5 * (g.t_lo + g.t_hi);
  gp.th = 0.5 * (g.t_hi - g.t_lo);
  gp.M = c->M;
  gp.jitter = c->sampling == DINR_JITTER;
  gp.seed_lo = (uint32_t)c->seed;
  gp.seed_hi = (uint32_t)(c->seed >> 32);
  gp.step = c->step;
  gp.ir = 1.0 / gp.r;
  gp.izh = gp.zh > 0.0 ? 1.0 / gp.zh : 0.0;
  gp.inv_sub_x = 1.0 / (double)gp.sub_x;
  gp.inv_sub_z = 1.0 / (double)gp.sub_z;
  gp.inv_ns = 1.0 / (double)gp.n_s;
  return gp;
}

template <class K>
dinr_status set_smem(dinr_ctx *c, K kernel, size_t bytes) {
  CUDA_TRY(c, cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return DINR_OK;
}

dinr_status launch_rays(dinr_ctx *c, const int64_t *idx, int64_t n, double *rec64, float4 *rec32, uint2 *rid,
                        cudaStream_t st, float *wq = nullptr) {
  if (n == 0) return DINR_OK;
  int64_t threads = n * c->S;
  Launch L_(c, T_RAYS, st);
  k_ray_setup<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(geom_params(c), c->d_views, idx, n, rec64, rec32,
                                                                  rid, c->d_flags, wq);
  CUDA_TRY(c, cudaGetLastError());
  return DINR_OK;
}

template <int H>
dinr_status launch_tc_mlp(dinr_ctx *c, const Plan &pl, int mode, cudaStream_t st) {
  TcParams p{};
  p.jit = pl.jit;
  p.rec32 = pl.rec32;
  p.nsamp = pl.nsamp;
  p.n_s = c->geom.samples_per_ray;
  p.L = c->L;
  p.resident = tc_resident(H, c->L) ? 1 : 0;
  p.mu0 = (float)c->field.mu0;
  p.params = c->d_params;
  p.B = c->d_B;
  p.wpack = c->d_wpack;
  p.pchunk = pl.pchunk;
  p.u = pl.u;
  p.hstash = pl.hstash;
  p.dstash = pl.dstash;
  p.zstash = pl.zstash;
  p.head_part = pl.head_part;
  p.n_tiles = pl.n_tiles;
  p.stash_feat = pl.feat0 ? 0 : 1;
  p.zall = pl.zall ? 1 : 0;
  p.db3 = pl.db3;
  size_t smem = TcLayout<H>::smem_bytes(c->L, p.resident != 0);
  if (mode == 2 && H == 256 && !pl.zall && fwd3_on() && !std::getenv("DINR_NO_BWD3") && !std::getenv("DINR_BWD2")) {
    // CTA pairs (cta_group::2, M = 256), two tile streams sharing each W_l block (k_tc_bwd3.cuh)
    const size_t sm3 = Bwd3Layout::smem_bytes();
    dinr_status s = set_smem(c, k_tc_bwd3, sm3);
    if (s) return s;
    const int clusters = (int)std::max<int64_t>(1, std::min<int64_t>(pl.n_tiles / 4, c->sm_count / 2));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * clusters), 1, 1);
    cfg.blockDim = dim3(Bwd3Layout::NT, 1, 1);
    cfg.dynamicSmemBytes = sm3;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    Launch L_(c, T_BWD, st);
    CUDA_TRY(c, cudaLaunchKernelEx(&cfg, k_tc_bwd3, p, pl.grid_tc));
  } else if (mode == 2 && H == 256 && !pl.zall && std::getenv("DINR_BWD2")) {
    // experiment (off by default: measured slower than k_tc_mlp MODE 2, which is HBM-bound, not
    // weight-load-bound): two tile streams per CTA, W_l streamed in halves shared by both
    const size_t sm2 = Bwd2Layout::smem_bytes();
    dinr_status s = set_smem(c, k_tc_bwd2, sm2);
    if (s) return s;
    Launch L_(c, T_BWD, st);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(pl.n_tiles / 2, c->sm_count));
    k_tc_bwd2<<<grid, Bwd2Layout::NT, sm2, st>>>(p, pl.grid_tc);
  } else if (mode == 2 && pl.zall) {
    dinr_status s = set_smem(c, k_tc_mlp<H, 3>, smem);
    if (s) return s;
    Launch L_(c, T_BWD, st);
    k_tc_mlp<H, 3><<<pl.grid_tc, kTcThreads, smem, st>>>(p);
  } else if (mode == 2) {
    dinr_status s = set_smem(c, k_tc_mlp<H, 2>, smem);
    if (s) return s;
    Launch L_(c, T_BWD, st);
    k_tc_mlp<H, 2><<<pl.grid_tc, kTcThreads, smem, st>>>(p);
  } else if (mode == 1 && H == 256 && fwd3_on() && Fwd3Layout::smem_bytes(c->L) <= kMaxSmem) {
    // CTA pairs (cta_group::2, M = 256), two tile streams, W_l through a ring of K-half buffers (k_tc_fwd3.cuh)
    const size_t sm3 = Fwd3Layout::smem_bytes(c->L);
    dinr_status s = set_smem(c, k_tc_fwd3, sm3);
    if (s) return s;
    const int clusters = (int)std::max<int64_t>(1, std::min<int64_t>(pl.n_tiles / 4, c->sm_count / 2));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * clusters), 1, 1);
    cfg.blockDim = dim3(Fwd3Layout::NT, 1, 1);
    cfg.dynamicSmemBytes = sm3;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
#ifdef DINR_PHASES
    static unsigned long long *dbg3 = nullptr;
    if (!dbg3) cudaMalloc(&dbg3, sizeof(unsigned long long) * 32 * 1024);
    cudaMemsetAsync(dbg3, 0, sizeof(unsigned long long) * 32 * 1024, st);
    p.dbg = dbg3;
#endif
    {
      Launch L_(c, T_FWD, st);
      CUDA_TRY(c, cudaLaunchKernelEx(&cfg, k_tc_fwd3, p));
    }
#ifdef DINR_PHASES
    {
      std::vector<unsigned long long> h((size_t)2 * clusters * 32);
      cudaStreamSynchronize(st);
      cudaMemcpy(h.data(), dbg3, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost);
      double tot[16] = {0};
      for (int b = 0; b < 2 * clusters; ++b)
        for (int k = 0; k < 16; ++k) tot[k] += (double)h[(size_t)b * 32 + k];
      const double it = (double)(pl.n_tiles / 4) * 2.0;  // CTA-iterations (both CTAs of every cluster)
      std::fprintf(stderr, "[fwd3 phases] cycles per CTA-iteration: s0 feat %.0f accwait %.0f epi %.0f | s1 feat %.0f "
                           "accwait %.0f epi %.0f | mma wait_w %.0f wait_a %.0f | loader wait_free %.0f wait_own %.0f | "
                           "store wait_a %.0f wait_read %.0f\n",
                   tot[0] / it, tot[1] / it, tot[2] / it, tot[4] / it, tot[5] / it, tot[6] / it, 2 * tot[8] / it,
                   2 * tot[9] / it, tot[10] / it, 2 * tot[11] / it, tot[12] / it, tot[13] / it);
    }
#endif
  } else if (mode == 1 && H == 256 && !std::getenv("DINR_NO_FWD2") && Fwd2Layout::smem_bytes(c->L) <= kMaxSmem) {
    // two tile streams per CTA, W_l streamed in N-halves (k_tc_fwd2.cuh)
    const size_t sm2 = Fwd2Layout::smem_bytes(c->L);
    dinr_status s = set_smem(c, k_tc_fwd2, sm2);
    if (s) return s;
    Launch L_(c, T_FWD, st);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(pl.n_tiles / 2, c->sm_count));
    k_tc_fwd2<<<grid, Fwd2Layout::NT, sm2, st>>>(p);
  } else if (mode == 1) {
    dinr_status s = set_smem(c, k_tc_mlp<H, 1>, smem);
    if (s) return s;
    Launch L_(c, T_FWD, st);
    k_tc_mlp<H, 1><<<pl.grid_tc, kTcThreads, smem, st>>>(p);
  } else {
    dinr_status s = set_smem(c, k_tc_mlp<H, 0>, smem);
    if (s) return s;
    Launch L_(c, T_FWD, st);
    k_tc_mlp<H, 0><<<pl.grid_tc, kTcThreads, smem, st>>>(p);
  }
  CUDA_TRY(c, cudaGetLastError());
  return DINR_OK;
}

template <int H>
dinr_status launch_tc_dw(dinr_ctx *c, const Plan &pl, cudaStream_t st) {
  DwParams p{};
  p.jit = pl.jit;
  p.hstash = pl.hstash;
  p.dstash = pl.dstash;
  p.n_tiles = pl.n_tiles;
  p.L = c->L;
  p.ksplit = pl.ksplit;
  p.nmb = pl.nmb;
  p.dw_part = pl.dw_part;
  p.db_part = pl.db_part;
  p.feat0 = pl.feat0 ? 1 : 0;  // layer 0's input (GRFF features) recomputed, not stashed
  p.ystash = pl.zstash;  // k_tc_dwz: inputs of layers >= 1 rebuilt from the y stash
  p.rec32 = pl.rec32;
  p.B = c->d_B;
  p.n_s = c->geom.samples_per_ray;
  p.lg_ns = 0;
  while ((1 << p.lg_ns) < p.n_s) ++p.lg_ns;
  p.nsamp = pl.nsamp;
  p.ks0 = pl.ks0;
  p.ks1 = pl.ks1;
  if (H == 256 && pl.zall) {
    const size_t smz = DwzLayout::smem_bytes();
    dinr_status s = set_smem(c, k_tc_dwz, smz);
    if (s) return s;
    Launch L_(c, T_DW, st);
    k_tc_dwz<<<dim3(pl.dw_layers * pl.ks1, 1, 1), DwzLayout::NT, smz, st>>>(p);
    CUDA_TRY(c, cudaGetLastError());
    return DINR_OK;
  }
  size_t smem = DwLayout<H>::smem_bytes();
  dinr_status s = set_smem(c, k_tc_dw<H>, smem);
  if (s) return s;
  Launch L_(c, T_DW, st);
  k_tc_dw<H><<<dim3(pl.ks0 + (pl.dw_layers - 1) * pl.ks1, pl.nmb, 1), DwLayout<H>::NT, smem, st>>>(p);
  CUDA_TRY(c, cudaGetLastError());
  return DINR_OK;
}

template <int H>
dinr_status launch_fused(dinr_ctx *c, const Plan &pl, const float *y, cudaStream_t st) {
  FusedParams p{};
  p.jit = pl.jit;
  p.rec32 = pl.rec32;
  p.n_pix = pl.n;
  p.nsamp = pl.nsamp;
  p.n_s = c->geom.samples_per_ray;
  p.lg_ns = 0;
  while ((1 << p.lg_ns) < p.n_s) ++p.lg_ns;
  p.S = c->S;
  p.L = c->L;
  p.nf = pl.nf;
  p.combine = c->field.combine;
  p.mu0 = (float)c->field.mu0;
  p.inv_n = 1.f / (float)pl.n;
  p.params = c->d_params;
  p.B = c->d_B;
  p.wpack_half = c->d_wpack_half;
  p.y = y;
  p.fhat = nullptr;  // training needs only the loss and u: no per-pixel projection store on the join
  p.ring = pl.ring;
  p.dw01 = pl.dw01 ? 1 : 0;
  p.hstash = pl.hstash;
  p.dstash = pl.dstash;
  p.n_tiles = pl.n_tiles;
  p.dw_part = pl.dwf;
  p.db_part = pl.dbf;
  p.head_part = pl.head_part;
  p.loss_part = pl.loss_part;
  const size_t smem = pl.fused2 ? Fused2Layout<H>::smem_bytes(c->L) : FusedLayout<H>::smem_bytes(c->L);
  dinr_status s = pl.fused2 ? set_smem(c, k_fused2<H>, smem) : set_smem(c, k_fused<H>, smem);
  if (s) return s;
#ifdef DINR_PHASES
  static unsigned long long *dbg = nullptr;
  if (!dbg) cudaMalloc(&dbg, sizeof(unsigned long long) * 8 * 1024);
  cudaMemsetAsync(dbg, 0, sizeof(unsigned long long) * 8 * 1024, st);
  p.dbg = dbg;
#endif
  {
    Launch L_(c, T_BWD, st);
    if (pl.fused2)
      k_fused2<H><<<pl.grid_f, Fused2Layout<H>::NT, smem, st>>>(p);
    else
      k_fused<H><<<pl.grid_f, FusedLayout<H>::NT, smem, st>>>(p);
  }
  CUDA_TRY(c, cudaGetLastError());
#ifdef DINR_PHASES
  if (pl.fused2) {
    std::vector<unsigned long long> h((size_t)pl.grid_f * 32);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), dbg, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost);
    const double groups = (double)((pl.nsamp + 255) / 256);
    for (int s = 0; s < 2; ++s) {
      double tot[9] = {0};
      for (int b = 0; b < pl.grid_f; ++b)
        for (int k = 0; k < 9; ++k) tot[k] += (double)h[(size_t)b * 32 + s * 16 + k];
      std::fprintf(stderr, "[dinr phases] stream %d cycles per group: feat %.0f fwd_wait %.0f fwd_epi %.0f loss %.0f "
                           "bwd_wait %.0f bwd_epi %.0f bwd_db %.0f end_wait %.0f (wait_sa %.0f)\n",
                   s, tot[0] / groups, tot[1] / groups, tot[2] / groups, tot[3] / groups, tot[4] / groups,
                   tot[5] / groups, tot[6] / groups, tot[7] / groups, tot[8] / groups);
    }
  } else {
    std::vector<unsigned long long> h((size_t)pl.grid_f * 8);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), dbg, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost);
    double tot[8] = {0};
    for (int b = 0; b < pl.grid_f; ++b)
      for (int k = 0; k < 8; ++k) tot[k] += (double)h[(size_t)b * 8 + k];
    const double tiles = (double)pl.n_tiles;
    std::fprintf(stderr, "[dinr phases] cycles per tile (CTA-avg): feat %.0f fwd_epi %.0f fwd_wait %.0f last+loss %.0f "
                         "bwd_epi %.0f bwd_wait %.0f bwd_pre %.0f\n",
                 tot[0] / tiles, tot[2] / tiles, tot[1] / tiles, tot[3] / tiles, tot[4] / tiles, tot[5] / tiles,
                 tot[6] / tiles);
  }
#endif
  return DINR_OK;
}

dinr_status tc_forward(dinr_ctx *c, const Plan &pl, int mode, cudaStream_t st) {
  switch (c->H) {
    case 64: return launch_tc_mlp<64>(c, pl, mode, st);
    case 128: return launch_tc_mlp<128>(c, pl, mode, st);
    case 256: return launch_tc_mlp<256>(c, pl, mode, st);
  }
  return fail(c, DINR_EINVAL, "unsupported width");
}

dinr_status launch_dw01(dinr_ctx *c, const Plan &pl, cudaStream_t st) {
  Dw01Params p{};
  p.dstash = pl.dstash;
  p.n_tiles = pl.n_tiles;
  p.nsamp = pl.nsamp;
  p.rec32 = pl.rec32;
  p.jit = pl.jit;
  p.B = c->d_B;
  p.n_s = c->geom.samples_per_ray;
  p.lg_ns = 0;
  while ((1 << p.lg_ns) < p.n_s) ++p.lg_ns;
  p.params = c->d_params;
  p.wpack_half = c->d_wpack_half;
  p.dw_part = pl.dw_part;
  p.db_part = pl.db_part;
  const size_t smem = Dw01Layout<128>::smem_bytes();
  dinr_status s = set_smem(c, k_dw01<128>, smem);
  if (s) return s;
  Launch L_(c, T_DW, st);
  k_dw01<128><<<pl.ksplit, Dw01Layout<128>::NT, smem, st>>>(p);
  CUDA_TRY(c, cudaGetLastError());
  return DINR_OK;
}

dinr_status tc_dw(dinr_ctx *c, const Plan &pl, cudaStream_t st) {
  if (pl.dw01) return launch_dw01(c, pl, st);
  switch (c->H) {
    case 64: return launch_tc_dw<64>(c, pl, st);
    case 128: return launch_tc_dw<128>(c, pl, st);
    case 256: return launch_tc_dw<256>(c, pl, st);
  }
  return fail(c, DINR_EINVAL, "unsupported width");
}

// ---------------------------------------------------------------- fp32 SIMT verify path
dinr_status simt_gemm(dinr_ctx *c, const SgemmArgs &a, int splits, cudaStream_t st, int cls) {
  dim3 grid((unsigned)((a.N + 63) / 64), (unsigned)((a.M + 63) / 64), (unsigned)splits);
  Launch L_(c, cls, st);
  s_gemm<<<grid, 256, 0, st>>>(a);
  CUDA_TRY(c, cudaGetLastError());
  return DINR_OK;
}

dinr_status simt_forward(dinr_ctx *c, const Plan &pl, cudaStream_t st) {
  const int H = c->H, L = c->L;
  const int64_t ns = pl.nsamp;
  {
    Launch L_(c, T_FWD, st);
    s_features<<<(unsigned)((ns + 255) / 256), 256, 0, st>>>(pl.rec32, ns, c->geom.samples_per_ray, c->d_B, c->C,
                                                           pl.sh, pl.jit);
  }
  CUDA_TRY(c, cudaGetLastError());
  const int64_t per = (int64_t)H * H + H;
  for (int l = 0; l < L; ++l) {
    SgemmArgs a{};
    a.A = pl.sh + (size_t)l * ns * H;
    a.sam = H;
    a.sak = 1;
    a.B = c->d_params + l * per;  // B(k=i, n=o) = W[o][i]
    a.sbk = 1;
    a.sbn = H;
    a.M = ns;
    a.N = H;
    a.K = H;
    a.kchunk = H;
    a.mode = 1;
    a.ldc = H;
    a.bias = c->d_params + l * per + (int64_t)H * H;
    a.Z = pl.sz + (size_t)l * ns * H;
    a.Hout = pl.sh + (size_t)(l + 1) * ns * H;
    dinr_status s = simt_gemm(c, a, 1, st, T_FWD);
    if (s) return s;
  }
  {
    Launch L_(c, T_FWD, st);
    s_head<<<(unsigned)((ns + 255) / 256), 256, 0, st>>>(pl.sh + (size_t)L * ns * H, ns, H,
                                                       c->d_params + L * per, (float)c->field.mu0,
                                                       pl.smu ? nullptr : pl.pchunk, pl.smu);
  }
  if (pl.smu) {  // N_s not a multiple of 32: per-ray sums in fixed order
    Launch L_(c, T_FWD, st);
    s_raysum<<<(unsigned)((pl.n_rays + 255) / 256), 256, 0, st>>>(pl.smu, pl.n_rays, c->geom.samples_per_ray, pl.pchunk);
  }
  CUDA_TRY(c, cudaGetLastError());
  return DINR_OK;
}

dinr_status simt_backward(dinr_ctx *c, const Plan &pl, cudaStream_t st) {
  const int H = c->H, L = c->L, ks = pl.ksplit_simt;
  const int64_t ns = pl.nsamp, per = (int64_t)H * H + H;
  const int n_s = c->geom.samples_per_ray;
  const int64_t rows_per = (ns + ks - 1) / ks;
  const float *wo = c->d_params + L * per;
  // head partials: sum_rows u h_L and sum u
  {
    Launch L_(c, T_BWD, st);
    s_colsum<<<dim3((unsigned)((H + 1 + 127) / 128), ks), 128, 0, st>>>(pl.sh + (size_t)L * ns * H, ns, H, rows_per,
                                                                       pl.u, n_s, pl.head_part, H + 1, 128, 1);
  }
  // delta_L = u w_o * swish'(z_L)
  {
    Launch L_(c, T_BWD, st);
    s_delta<<<(unsigned)((ns * H + 255) / 256), 256, 0, st>>>(pl.sd, pl.sz + (size_t)(L - 1) * ns * H, ns, H, pl.u,
                                                            n_s, wo);
  }
  for (int l = L - 1; l >= 0; --l) {
    // dW_l = delta_l^T h_l (split-K partials into dw_part [l][mb][ks][128][H])
    SgemmArgs a{};
    a.A = pl.sd;
    a.sam = 1;
    a.sak = H;
    a.B = pl.sh + (size_t)l * ns * H;
    a.sbk = H;
    a.sbn = 1;
    a.M = H;
    a.N = H;
    a.K = ns;
    a.kchunk = rows_per;
    a.mode = 0;
    a.C = pl.dw_part + (size_t)l * pl.nmb * ks * 128 * H;
    a.ldc = H;
    a.cz = 128 * H;
    a.cmb = (int64_t)ks * 128 * H;
    dinr_status s = simt_gemm(c, a, ks, st, T_DW);
    if (s) return s;
    {
      Launch L_(c, T_DW, st);
      s_colsum<<<dim3((unsigned)((H + 127) / 128), ks), 128, 0, st>>>(
          pl.sd, ns, H, rows_per, nullptr, n_s, pl.db_part + (size_t)l * pl.nmb * ks * 128, 128, (int64_t)ks * 128, 0);
    }
    if (l > 0) {
      // e_{l-1} = delta_l W_l  (into the z buffer of layer l, which is no longer needed)
      float *e = pl.sz + (size_t)l * ns * H;
      SgemmArgs b{};
      b.A = pl.sd;
      b.sam = H;
      b.sak = 1;
      b.B = c->d_params + l * per;  // B(k=o, n=i) = W[o][i]
      b.sbk = H;
      b.sbn = 1;
      b.M = ns;
      b.N = H;
      b.K = H;
      b.kchunk = H;
      b.mode = 0;
      b.C = e;
      b.ldc = H;
      b.cz = 0;
      b.cmb = 128 * H;
      s = simt_gemm(c, b, 1, st, T_BWD);
      if (s) return s;
      {
        Launch L_(c, T_BWD, st);
        s_delta<<<(unsigned)((ns * H + 255) / 256), 256, 0, st>>>(e, pl.sz + (size_t)(l - 1) * ns * H, ns, H,
                                                                nullptr, n_s, nullptr);
      }
      CUDA_TRY(c, cudaMemcpyAsync(pl.sd, e, sizeof(float) * ns * H, cudaMemcpyDeviceToDevice, st));
    }
  }
  CUDA_TRY(c, cudaGetLastError());
  return DINR_OK;
}

dinr_status run_loss(dinr_ctx *c, const Plan &pl, const float *y, float *fhat, float *p_sub, const float *I0,
                     float *Ihat, cudaStream_t st) {
  if (pl.n == 0) return DINR_OK;
  Launch L_(c, T_LOSS, st);
  k_loss<<<pl.nloss, kLossThreads, 0, st>>>(pl.wq, pl.pchunk, c->S, pl.nc, pl.n, y, c->field.combine,
                                            (float)c->field.mu0, fhat, p_sub, I0, Ihat, pl.u,
                                            y ? pl.loss_part : nullptr);
  CUDA_TRY(c, cudaGetLastError());
  return DINR_OK;
}

dinr_status step_grad(dinr_ctx *c, const int64_t *idx, int64_t n, const float *y, float *grad, int accumulate,
                      Plan &pl, cudaStream_t st) {
  dinr_status s;
  if (n == 0) {
    if (!accumulate) CUDA_TRY(c, cudaMemsetAsync(grad, 0, sizeof(float) * (c->P + 1), st));
    return DINR_OK;
  }
  s = launch_rays(c, idx, n, nullptr, pl.rec32, pl.jit.rid ? pl.rid : nullptr, st, pl.wq);
  if (s) return s;
  if (pl.fused) {
    s = c->H == 64 ? launch_fused<64>(c, pl, y, st) : launch_fused<128>(c, pl, y, st);
    if (s) return s;
    if (pl.nu > 0) {
      s = tc_dw(c, pl, st);
      if (s) return s;
    }
    Launch L_(c, T_ASM, st);
    k_assemble2<<<(unsigned)((c->P + 1 + 31) / 32), 256, 0, st>>>(
        c->H, c->L, c->P, pl.nu, pl.ksplit, pl.dw_part, pl.db_part, pl.grid_f, pl.dwf, pl.dbf, pl.head_part,
        pl.grid_f, pl.loss_part, pl.grid_f, 1.f / (float)n, accumulate, grad);
    CUDA_TRY(c, cudaGetLastError());
    return DINR_OK;
  }
  const bool simt = c->field.precision == DINR_FP32_VERIFY;
  if (simt) {
    s = simt_forward(c, pl, st);
  } else {
    s = tc_forward(c, pl, 1, st);  // training forward: stashes h_l and z_l for K3 / K5
  }
  if (s) return s;
  s = run_loss(c, pl, y, pl.fhat, nullptr, nullptr, nullptr, st);
  if (s) return s;
  int nhead, ks;
  if (simt) {
    s = simt_backward(c, pl, st);
    nhead = pl.ksplit_simt;
    ks = pl.ksplit_simt;
  } else {
    s = tc_forward(c, pl, 2, st);  // backward from the stashes
    if (s) return s;
    s = tc_dw(c, pl, st);
    nhead = pl.grid_tc;
    ks = pl.ksplit;
  }
  if (s) return s;
  {
    Launch L_(c, T_ASM, st);
    k_assemble<<<(unsigned)((c->P + 1 + 255) / 256), 256, 0, st>>>(
        c->H, c->L, c->P, pl.nmb, ks, pl.dw_part, pl.zall ? pl.db3 : pl.db_part, pl.zall ? pl.grid_tc : ks,
        pl.head_part, nhead, pl.loss_part, pl.nloss, 1.f / (float)n, accumulate, grad);
  }
  CUDA_TRY(c, cudaGetLastError());
  return DINR_OK;
}

}  // namespace

extern "C" {

int64_t dinr_param_count(int32_t n_freq, int32_t n_layers) {
  int64_t H = 2 * (int64_t)n_freq;
  return (int64_t)n_layers * (H * H + H) + H + 1;
}

const char *dinr_status_string(dinr_status s) {
  switch (s) {
    case DINR_OK: return "DINR_OK";
    case DINR_EINVAL: return "DINR_EINVAL";
    case DINR_ERANGE: return "DINR_ERANGE";
    case DINR_ENOMEM: return "DINR_ENOMEM";
    case DINR_ECUDA: return "DINR_ECUDA";
    case DINR_ENCCL: return "DINR_ENCCL";
    case DINR_ESTATE: return "DINR_ESTATE";
    case DINR_EDEVICE: return "DINR_EDEVICE";
  }
  return "DINR_UNKNOWN";
}

dinr_status dinr_create(int device, dinr_ctx **out) {
  if (!out) return DINR_EINVAL;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return DINR_EDEVICE;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major != 10) return DINR_EDEVICE;
  dinr_ctx *c = new (std::nothrow) dinr_ctx();
  if (!c) return DINR_ENOMEM;
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  if (cudaSetDevice(device) != cudaSuccess || cudaMalloc(&c->d_flags, 16) != cudaSuccess ||
      cudaMemset(c->d_flags, 0, 16) != cudaSuccess) {
    delete c;
    return DINR_ECUDA;
  }
  *out = c;
  return DINR_OK;
}

dinr_status dinr_destroy(dinr_ctx *c) {
  if (!c) return DINR_EINVAL;
  cudaSetDevice(c->device);
  for (auto &p : c->pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : c->event_pool) cudaEventDestroy(e);
  if (c->comm) nccl().CommDestroy((ncclComm_t)c->comm);
  cudaFree(c->d_views);
  cudaFree(c->d_B);
  cudaFree(c->d_params);
  cudaFree(c->d_wpack);
  cudaFree(c->d_wpack_half);
  cudaFree(c->d_prims);
  cudaFree(c->scratch);
  cudaFree(c->d_flags);
  delete c;
  return DINR_OK;
}

const char *dinr_last_error(const dinr_ctx *c) { return c ? c->err.c_str() : "null context"; }

dinr_status dinr_set_sampling(dinr_ctx *c, dinr_sampling mode, uint64_t seed, uint32_t step) {
  if (!c) return DINR_EINVAL;
  if (mode != DINR_MIDPOINT && mode != DINR_JITTER) return fail(c, DINR_EINVAL, "unknown sampling mode");
  c->sampling = mode;
  c->seed = seed;
  c->step = step;
  return DINR_OK;
}

dinr_status dinr_set_geometry(dinr_ctx *c, const dinr_geometry *g_in, const double *theta, const double *t, int64_t M) {
  if (!c || !g_in || !theta || !t) return c ? fail(c, DINR_EINVAL, "null argument") : DINR_EINVAL;
  // NaN normalization ranges are derived (R11): detector z extent (cone: scaled to the far side of
  // the FOV cylinder), first / last view time
  dinr_geometry gd = *g_in;
  if (std::isnan(gd.z_lo) || std::isnan(gd.z_hi)) {
    double zlo = -gd.offset_cz, zhi = -gd.offset_cz + (double)gd.n_rows * gd.pixel_dz;
    if (gd.beam == DINR_CONE) {
      const double mag_far = (gd.sod + gd.fov_radius) / (gd.sod + gd.odd);
      zlo *= mag_far;
      zhi *= mag_far;
    }
    if (std::isnan(gd.z_lo)) gd.z_lo = zlo;
    if (std::isnan(gd.z_hi)) gd.z_hi = zhi;
  }
  if (M >= 1 && (std::isnan(gd.t_lo) || std::isnan(gd.t_hi))) {
    if (std::isnan(gd.t_lo)) gd.t_lo = t[0];
    if (std::isnan(gd.t_hi)) gd.t_hi = t[M - 1];
  }
  const dinr_geometry *g = &gd;
  if (g->beam < 0 || g->beam > 2) return fail(c, DINR_EINVAL, "beam must be 0 (parallel), 1 (fan) or 2 (cone)");
  if (g->n_rows < 1 || g->n_cols < 1) return fail(c, DINR_EINVAL, "n_rows, n_cols must be >= 1");
  if (g->sub_x < 1 || g->sub_z < 1 || g->sub_x * g->sub_z > kMaxS)
    return fail(c, DINR_EINVAL, "sub_x, sub_z must be >= 1 with sub_x*sub_z <= 16");
  // N_s: any N_s >= 1 on the fp32 verify path; a multiple of 32 on the bf16 tensor-core path (the
  // performance contract: a ray is whole warps), checked here when the weights are already set and
  // by dinr_set_field_weights otherwise
  if (g->samples_per_ray < 1) return fail(c, DINR_EINVAL, "samples_per_ray must be >= 1");
  if (c->have_field && c->field.precision == DINR_BF16 && g->samples_per_ray % 32)
    return fail(c, DINR_EINVAL, "the BF16 path needs samples_per_ray a multiple of 32 (FP32_VERIFY accepts any)");
  const double v[] = {g->sod, g->odd, g->pixel_dx, g->pixel_dz, g->offset_cx, g->offset_cz, g->fov_radius,
                      g->rot_center_x, g->z_lo, g->z_hi, g->t_lo, g->t_hi};
  for (double x : v)
    if (!is_fin(x)) return fail(c, DINR_EINVAL, "geometry values must be finite");
  if (!(g->sod > 0) || !(g->odd >= 0) || !(g->pixel_dx > 0) || !(g->pixel_dz > 0) || !(g->fov_radius > 0))
    return fail(c, DINR_EINVAL, "need sod > 0, odd >= 0, pixel pitches > 0, fov_radius > 0 (S:24-27)");
  if (!(g->fov_radius < g->sod)) return fail(c, DINR_EINVAL, "fov_radius must be < sod (source outside the FOV)");
  if (!(g->z_hi >= g->z_lo) || !(g->t_hi >= g->t_lo)) return fail(c, DINR_EINVAL, "normalization ranges inverted");
  if (M < 1) return fail(c, DINR_EINVAL, "M must be >= 1");
  for (int64_t k = 0; k < M; ++k) {
    if (!is_fin(theta[k]) || !is_fin(t[k])) return fail(c, DINR_EINVAL, "non-finite view angle or time");
    if (k > 0 && t[k] < t[k - 1]) return fail(c, DINR_EINVAL, "view times must be non-decreasing");
  }
  std::vector<double> tab((size_t)M * 3);
  for (int64_t k = 0; k < M; ++k) {  // host libm, same as the oracle (O1)
    tab[3 * k] = std::cos(theta[k]);
    tab[3 * k + 1] = std::sin(theta[k]);
    tab[3 * k + 2] = t[k];
  }
  CUDA_TRY(c, cudaSetDevice(c->device));
  double *dv = nullptr;
  CUDA_TRY(c, cudaMalloc(&dv, sizeof(double) * tab.size()));
  if (cudaMemcpy(dv, tab.data(), sizeof(double) * tab.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(dv);
    return fail(c, DINR_ECUDA, "view table upload failed");
  }
  cudaFree(c->d_views);
  c->d_views = dv;
  c->geom = *g;
  c->M = M;
  c->S = g->sub_x * g->sub_z;
  c->h_t.assign(t, t + M);
  c->have_geom = true;
  return DINR_OK;
}

dinr_status dinr_set_field_weights(dinr_ctx *c, const dinr_field_desc *f, const float *B_dev, const float *params_dev,
                                   void *stream) {
  if (!c || !f || !B_dev || !params_dev) return c ? fail(c, DINR_EINVAL, "null argument") : DINR_EINVAL;
  if (!c->have_geom) return fail(c, DINR_ESTATE, "dinr_set_geometry must be called first");
  if (f->n_freq < 1 || f->width != 2 * f->n_freq || f->n_layers < 1 || f->n_layers > 64)
    return fail(c, DINR_EINVAL, "need n_freq >= 1, width == 2*n_freq, 1 <= n_layers <= 64");
  if (!(f->mu0 > 0) || !is_fin(f->mu0)) return fail(c, DINR_EINVAL, "mu0 must be > 0");
  if (f->combine != DINR_BEER && f->combine != DINR_LINEAR) return fail(c, DINR_EINVAL, "bad combine");
  if (f->precision == DINR_BF16) {
    if (f->width != 64 && f->width != 128 && f->width != 256)
      return fail(c, DINR_EINVAL, "BF16 path supports width 64, 128 or 256");
    if (c->geom.samples_per_ray % 32)
      return fail(c, DINR_EINVAL, "the BF16 path needs samples_per_ray a multiple of 32 (FP32_VERIFY accepts any)");
    // at H = 256 every layer's bias sits in the tensor-core kernels' shared memory
    if (f->width == 256 && TcLayout<256>::smem_bytes(f->n_layers, false) > kMaxSmem)
      return fail(c, DINR_EINVAL, "the BF16 path supports n_layers <= 27 at width 256");
  } else if (f->precision == DINR_FP32_VERIFY) {
    if (f->width > kMaxH || f->width % 2) return fail(c, DINR_EINVAL, "FP32_VERIFY supports width <= 256");
  } else {
    return fail(c, DINR_EINVAL, "bad precision");
  }
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(c, cudaSetDevice(c->device));
  const int H = f->width, L = f->n_layers;
  const int64_t P = dinr_param_count(f->n_freq, f->n_layers);
  size_t pbytes = sizeof(float) * (P + 4);
  if (pbytes > c->params_cap) {
    cudaFree(c->d_params);
    c->d_params = nullptr;
    CUDA_TRY(c, cudaMalloc(&c->d_params, pbytes));
    c->params_cap = pbytes;
  }
  size_t wbytes = (size_t)L * H * H * 2;
  if (wbytes > c->wpack_cap) {
    cudaFree(c->d_wpack);
    cudaFree(c->d_wpack_half);
    c->d_wpack = c->d_wpack_half = nullptr;
    c->wpack_cap = 0;
    CUDA_TRY(c, cudaMalloc(&c->d_wpack, wbytes));
    CUDA_TRY(c, cudaMalloc(&c->d_wpack_half, wbytes));
    c->wpack_cap = wbytes;
  }
  if (!c->d_B || f->n_freq > c->C) {
    cudaFree(c->d_B);
    c->d_B = nullptr;
    CUDA_TRY(c, cudaMalloc(&c->d_B, sizeof(float) * 4 * std::max(f->n_freq, kMaxH / 2)));
  }
  CUDA_TRY(c, cudaMemcpyAsync(c->d_B, B_dev, sizeof(float) * 4 * f->n_freq, cudaMemcpyDeviceToDevice, st));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_params, params_dev, sizeof(float) * P, cudaMemcpyDeviceToDevice, st));
  c->field = *f;
  c->C = f->n_freq;
  c->L = L;
  c->H = H;
  c->P = P;
  if (f->precision == DINR_BF16) {
    Launch L_(c, T_PACK, st);
    int64_t tot = (int64_t)L * H * H;
    k_pack_weights<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(c->d_params, H, L, c->d_wpack, c->d_wpack_half);
  }
  CUDA_TRY(c, cudaGetLastError());
  c->have_field = true;
  return DINR_OK;
}

dinr_status dinr_adam_step(dinr_ctx *c, float *params, const float *grad, float *m, float *v, int64_t count,
                           double lr, double b1, double b2, double eps, int64_t step, void *stream) {
  if (!c) return DINR_EINVAL;
  if (!c->have_field) return fail(c, DINR_ESTATE, "dinr_set_field_weights must be called first");
  if (!params || !grad || !m || !v || count != c->P || step < 1 || !(lr >= 0) || !(b1 >= 0 && b1 < 1) ||
      !(b2 >= 0 && b2 < 1) || !(eps > 0))
    return fail(c, DINR_EINVAL, "bad Adam arguments (count must equal P, step >= 1, 0 <= beta < 1, eps > 0)");
  CUDA_TRY(c, cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  const float c1 = (float)(1.0 - std::pow(b1, (double)step)), c2 = (float)(1.0 - std::pow(b2, (double)step));
  const bool bf16 = c->field.precision == DINR_BF16;  // FP32_VERIFY widths need not be multiples of 64
  Launch L_(c, T_PACK, st);
  k_adam_pack<<<(unsigned)((c->P + 255) / 256), 256, 0, st>>>(params, grad, m, v, c->P, c->H, c->L, (float)lr,
                                                              (float)b1, (float)b2, (float)eps, c1, c2, c->d_params,
                                                              bf16 ? c->d_wpack : nullptr,
                                                              bf16 ? c->d_wpack_half : nullptr);
  CUDA_TRY(c, cudaGetLastError());
  return DINR_OK;
}

}  // extern "C"

namespace {

// N1: the validated shape of a dinr_train_desc for this context (see include/dinr.h)
dinr_status train_desc_check(dinr_ctx *c, const dinr_train_desc *d, int64_t *D, int64_t *ipe) {
  if (!d) return fail(c, DINR_EINVAL, "null train desc");
  if (!c->have_geom) return fail(c, DINR_ESTATE, "dinr_set_geometry must be called first");
  if (d->world < 1 || d->rank < 0 || d->rank >= d->world || d->batch < 1 ||
      (d->sharding != DINR_SHARD_VIEWS && d->sharding != DINR_SHARD_GLOBAL) || !(d->lr0 >= 0) ||
      !(d->lr_decay > 0) || !(d->beta1 >= 0 && d->beta1 < 1) || !(d->beta2 >= 0 && d->beta2 < 1) || !(d->eps > 0))
    return fail(c, DINR_EINVAL, "bad train desc (0 <= rank < world, batch >= 1, sharding, lr0 >= 0, lr_decay > 0, "
                                "0 <= beta < 1, eps > 0)");
  const int64_t N = (int64_t)c->geom.n_rows * c->geom.n_cols;
  if (d->sharding == DINR_SHARD_VIEWS) {
    const int64_t nv = (c->M - d->rank + d->world - 1) / d->world;
    if (nv < 1) return fail(c, DINR_EINVAL, "view sharding: more processes than views");
    *D = nv * N;
  } else {
    *D = c->M * N;
  }
  const int64_t per = (int64_t)d->world * d->batch;
  *ipe = (c->M * N + per - 1) / per;
  return DINR_OK;
}

dinr_status launch_sample(dinr_ctx *c, const dinr_train_desc *d, int64_t D, int64_t epoch, int64_t it,
                          const float *y_src, int64_t *idx, float *y, cudaStream_t st) {
  SampleArgs a;
  a.N = (int64_t)c->geom.n_rows * c->geom.n_cols;
  a.D = D;
  a.n = d->batch;
  // it * world * batch <= M N + world * batch for any iteration of an epoch; the caller's
  // iteration index is reduced mod the shard first, so the sum cannot overflow
  const int64_t per = d->sharding == DINR_SHARD_VIEWS ? d->batch : (int64_t)d->world * d->batch;
  const int64_t off = d->sharding == DINR_SHARD_VIEWS ? 0 : (int64_t)d->rank * d->batch;
  a.base = (int64_t)(((unsigned __int128)(uint64_t)it * (uint64_t)per + (uint64_t)off) % (uint64_t)D);
  int h = 1;
  while ((1ull << (2 * h)) < (uint64_t)D) ++h;
  a.h = h;
  a.mode = d->sharding;
  a.rank = d->rank;
  a.world = d->world;
  a.key = make_uint2((uint32_t)d->seed, (uint32_t)(d->seed >> 32) ^ 0x9E3779B9u);
  a.e_lo = (uint32_t)epoch;
  a.e_hi = (uint32_t)((uint64_t)epoch >> 32);
  a.y_src = y_src;
  a.idx = idx;
  a.y = y;
  Launch L_(c, T_RAYS, st);
  k_sample_batch<<<(unsigned)((d->batch + 255) / 256), 256, 0, st>>>(a);
  CUDA_TRY(c, cudaGetLastError());
  return DINR_OK;
}

}  // namespace

extern "C" {

dinr_status dinr_iterations_per_epoch(dinr_ctx *c, const dinr_train_desc *d, int64_t *out) {
  if (!c || !out) return c ? fail(c, DINR_EINVAL, "null argument") : DINR_EINVAL;
  int64_t D, ipe;
  dinr_status s = train_desc_check(c, d, &D, &ipe);
  if (s) return s;
  *out = ipe;
  return DINR_OK;
}

dinr_status dinr_sample_batch(dinr_ctx *c, const dinr_train_desc *d, int64_t epoch, int64_t it, const float *y_src,
                              int64_t *idx, float *y, void *stream) {
  if (!c) return DINR_EINVAL;
  if (!idx || (y_src && !y) || epoch < 0 || it < 0) return fail(c, DINR_EINVAL, "bad arguments");
  int64_t D, ipe;
  dinr_status s = train_desc_check(c, d, &D, &ipe);
  if (s) return s;
  CUDA_TRY(c, cudaSetDevice(c->device));
  return launch_sample(c, d, D, epoch, it, y_src, idx, y, (cudaStream_t)stream);
}

dinr_status dinr_train_iterations(dinr_ctx *c, const dinr_train_desc *d, int64_t first, int64_t count,
                                  const float *y_src, float *params, float *m, float *v, float *grad, float *loss,
                                  void *stream) {
  if (!c) return DINR_EINVAL;
  if (!c->have_field) return fail(c, DINR_ESTATE, "dinr_set_field_weights must be called first");
  if (first < 0 || count < 0 || !y_src || !params || !m || !v || !grad || (count > 0 && !loss))
    return fail(c, DINR_EINVAL, "bad arguments");
  int64_t D, ipe;
  dinr_status s = train_desc_check(c, d, &D, &ipe);
  if (s) return s;
  if (d->world > 1 && (!c->comm || c->world != d->world || c->rank != d->rank))
    return fail(c, DINR_ESTATE, "world > 1 needs dinr_comm_init with the same rank and world");
  CUDA_TRY(c, cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  for (int64_t g = first; g < first + count; ++g) {
    const int64_t epoch = g / ipe, it = g % ipe;
    Plan pl;
    s = ensure_plan(c, d->batch, true, true, pl);  // host_io: the batch's idx / y buffers
    if (s) return s;
    s = launch_sample(c, d, D, epoch, it, y_src, pl.idx_dev, pl.y_dev, st);
    if (s) return s;
    s = step_grad(c, pl.idx_dev, d->batch, pl.y_dev, grad, 0, pl, st);
    if (s) return s;
    if (d->world > 1) {
      s = dinr_allreduce_grads(c, grad, c->P + 1, stream);
      if (s) return s;
    }
    CUDA_TRY(c, cudaMemcpyAsync(loss + (g - first), grad + c->P, sizeof(float), cudaMemcpyDeviceToDevice, st));
    s = dinr_adam_step(c, params, grad, m, v, c->P, d->lr0 * std::pow(d->lr_decay, (double)epoch), d->beta1,
                       d->beta2, d->eps, g + 1, stream);
    if (s) return s;
  }
  return DINR_OK;
}

dinr_status dinr_phantom_project(dinr_ctx *c, const dinr_primitive *prims, int32_t np, const int64_t *idx, int64_t n,
                                 int32_t combine, double noise_frac, uint64_t seed, float *fhat, float *p_sub,
                                 void *stream) {
  if (!c) return DINR_EINVAL;
  if (!c->have_geom) return fail(c, DINR_ESTATE, "dinr_set_geometry must be called first");
  if (np < 0 || np > 64 || (np > 0 && !prims) || n < 0 || (n > 0 && (!idx || !fhat)) ||
      (combine != DINR_BEER && combine != DINR_LINEAR) || !(noise_frac >= 0))
    return fail(c, DINR_EINVAL, "bad arguments (0 <= n_prims <= 64, combine, noise_frac >= 0)");
  std::vector<PrimDev> h((size_t)std::max(1, np));
  for (int q = 0; q < np; ++q) {
    if (prims[q].kind < 0 || prims[q].kind > 2) return fail(c, DINR_EINVAL, "primitive kind must be 0, 1 or 2");
    h[q].kind = prims[q].kind;
    h[q].value = prims[q].value;
    for (int k = 0; k < 3; ++k) {
      if (!(prims[q].axes[k] > 0)) return fail(c, DINR_EINVAL, "primitive axes must be > 0");
      h[q].c0[k] = prims[q].center[k];
      h[q].vel[k] = prims[q].velocity[k];
      h[q].a0[k] = prims[q].axes[k];
      h[q].arate[k] = prims[q].axes_rate[k];
    }
  }
  if (n == 0) return DINR_OK;
  CUDA_TRY(c, cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  if (!c->d_prims) CUDA_TRY(c, cudaMalloc(&c->d_prims, sizeof(PrimDev) * 64));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_prims, h.data(), sizeof(PrimDev) * np, cudaMemcpyHostToDevice, st));
  CUDA_TRY(c, cudaStreamSynchronize(st));  // the host staging vector dies with this call
  Launch L_(c, T_RAYS, st);
  k_phantom_project<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(geom_params(c), c->d_views, idx, n,
                                                                (const PrimDev *)c->d_prims, np, combine, noise_frac,
                                                                seed, fhat, p_sub, c->d_flags);
  CUDA_TRY(c, cudaGetLastError());
  return DINR_OK;
}

dinr_status dinr_ray_records(dinr_ctx *c, const int64_t *idx, int64_t n, double *rec, void *stream) {
  if (!c) return DINR_EINVAL;
  if (!c->have_geom) return fail(c, DINR_ESTATE, "dinr_set_geometry must be called first");
  if (n < 0 || (n > 0 && (!idx || !rec))) return fail(c, DINR_EINVAL, "bad arguments");
  CUDA_TRY(c, cudaSetDevice(c->device));
  return launch_rays(c, idx, n, rec, nullptr, nullptr, (cudaStream_t)stream);
}

dinr_status dinr_project(dinr_ctx *c, const int64_t *idx, int64_t n, float *fhat, float *p_sub, const float *I0,
                         float *Ihat, void *stream) {
  if (!c) return DINR_EINVAL;
  if (!c->have_geom || !c->have_field) return fail(c, DINR_ESTATE, "geometry and field weights must be set first");
  if (n < 0 || (n > 0 && (!idx || !fhat)) || ((I0 == nullptr) != (Ihat == nullptr)))
    return fail(c, DINR_EINVAL, "bad arguments");
  if (n == 0) return DINR_OK;
  CUDA_TRY(c, cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  Plan pl;
  dinr_status s = ensure_plan(c, n, false, false, pl);
  if (s) return s;
  s = launch_rays(c, idx, n, nullptr, pl.rec32, pl.jit.rid ? pl.rid : nullptr, st, pl.wq);
  if (s) return s;
  s = c->field.precision == DINR_FP32_VERIFY ? simt_forward(c, pl, st) : tc_forward(c, pl, 0, st);
  if (s) return s;
  return run_loss(c, pl, nullptr, fhat, p_sub, I0, Ihat, st);
}

dinr_status dinr_project_and_grad(dinr_ctx *c, const int64_t *idx, int64_t n, const float *y, float *grad,
                                  int accumulate, void *stream) {
  if (!c) return DINR_EINVAL;
  if (!c->have_geom || !c->have_field) return fail(c, DINR_ESTATE, "geometry and field weights must be set first");
  if (n < 0 || !grad || (n > 0 && (!idx || !y))) return fail(c, DINR_EINVAL, "bad arguments");
  CUDA_TRY(c, cudaSetDevice(c->device));
  Plan pl;
  dinr_status s = ensure_plan(c, n, true, false, pl);
  if (s) return s;
  return step_grad(c, idx, n, y, grad, accumulate, pl, (cudaStream_t)stream);
}

dinr_status dinr_project_and_grad_host(dinr_ctx *c, const int64_t *idx_host, int64_t n, const float *y_host,
                                       float *grad_host, int allreduce, void *stream) {
  if (!c) return DINR_EINVAL;
  if (!c->have_geom || !c->have_field) return fail(c, DINR_ESTATE, "geometry and field weights must be set first");
  if (n < 0 || !grad_host || (n > 0 && (!idx_host || !y_host))) return fail(c, DINR_EINVAL, "bad arguments");
  if (allreduce && !c->comm && c->world > 1) return fail(c, DINR_ESTATE, "communicator not initialized");
  CUDA_TRY(c, cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  Plan pl;
  dinr_status s = ensure_plan(c, n, true, true, pl);
  if (s) return s;
  if (n > 0) {
    CUDA_TRY(c, cudaMemcpyAsync(pl.idx_dev, idx_host, sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(c, cudaMemcpyAsync(pl.y_dev, y_host, sizeof(float) * n, cudaMemcpyHostToDevice, st));
  }
  s = step_grad(c, pl.idx_dev, n, pl.y_dev, pl.grad_dev, 0, pl, st);
  if (s) return s;
  if (allreduce && c->comm) {
    s = dinr_allreduce_grads(c, pl.grad_dev, c->P + 1, stream);
    if (s) return s;
  }
  CUDA_TRY(c, cudaMemcpyAsync(grad_host, pl.grad_dev, sizeof(float) * (c->P + 1), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(c, cudaStreamSynchronize(st));
  return DINR_OK;
}

dinr_status dinr_nccl_unique_id(void *out) {
  if (!out) return DINR_EINVAL;
  ncclUniqueId id;
  if (!nccl().ok || nccl().GetUniqueId(&id) != ncclSuccess) return DINR_ENCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
  std::memcpy(out, &id, sizeof(id));
  return DINR_OK;
}

dinr_status dinr_comm_init(dinr_ctx *c, const void *uid, int rank, int world) {
  if (!c || !uid || world < 1 || rank < 0 || rank >= world) return c ? fail(c, DINR_EINVAL, "bad rank/world") : DINR_EINVAL;
  if (!nccl().ok) return fail(c, DINR_ENCCL, nccl().err);
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (c->comm) {
    nccl().CommDestroy((ncclComm_t)c->comm);
    c->comm = nullptr;
  }
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof(id));
  ncclComm_t comm;
  ncclResult_t r = nccl().CommInitRank(&comm, world, id, rank);
  if (r != ncclSuccess) return fail(c, DINR_ENCCL, std::string("ncclCommInitRank: ") + nccl().GetErrorString(r));
  c->comm = comm;
  c->rank = rank;
  c->world = world;
  return DINR_OK;
}

dinr_status dinr_allreduce_grads(dinr_ctx *c, float *grad, int64_t count, void *stream) {
  if (!c || !grad || count < 0) return c ? fail(c, DINR_EINVAL, "bad arguments") : DINR_EINVAL;
  if (!c->comm) return fail(c, DINR_ESTATE, "dinr_comm_init must be called first");
  CUDA_TRY(c, cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  Launch L_(c, T_AR, st);
  ncclResult_t r = nccl().AllReduce(grad, grad, (size_t)count, ncclFloat32, ncclAvg, (ncclComm_t)c->comm, st);
  if (r != ncclSuccess) return fail(c, DINR_ENCCL, std::string("ncclAllReduce: ") + nccl().GetErrorString(r));
  return DINR_OK;
}

dinr_status dinr_get_device_status(dinr_ctx *c) {
  if (!c) return DINR_EINVAL;
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaDeviceSynchronize());
  int flags[1] = {0};
  CUDA_TRY(c, cudaMemcpy(flags, c->d_flags, sizeof(flags), cudaMemcpyDeviceToHost));
  CUDA_TRY(c, cudaMemset(c->d_flags, 0, sizeof(flags)));
  size_t bad = 0;
  if (guards_on() && !guards_intact(c, &bad))
    return fail(c, DINR_EDEVICE, "DINR_GUARDS: scratch guard band overwritten at byte " + std::to_string(bad));
  if (flags[0] & 1) return fail(c, DINR_ERANGE, "a pixel index was out of range (>= M*N); it contributed 0");
  return DINR_OK;
}

dinr_status dinr_set_timing(dinr_ctx *c, int enable) {
  if (!c) return DINR_EINVAL;
  c->timing = enable != 0;
  return DINR_OK;
}

dinr_status dinr_read_timing(dinr_ctx *c, int which, double *ms, int64_t *launches, int reset) {
  if (!c || which < 0 || which >= T_N) return c ? fail(c, DINR_EINVAL, "bad timer class") : DINR_EINVAL;
  for (auto &p : c->pending) {
    CUDA_TRY(c, cudaEventSynchronize(p.b));
    float e = 0.f;
    CUDA_TRY(c, cudaEventElapsedTime(&e, p.a, p.b));
    c->acc_ms[p.cls] += e;
    c->acc_n[p.cls] += 1;
    c->event_pool.push_back(p.a);
    c->event_pool.push_back(p.b);
  }
  c->pending.clear();
  if (ms) *ms = c->acc_ms[which];
  if (launches) *launches = c->acc_n[which];
  if (reset) {
    c->acc_ms[which] = 0;
    c->acc_n[which] = 0;
  }
  return DINR_OK;
}

int64_t dinr_launch_count(const dinr_ctx *c) { return c ? c->launches : 0; }

dinr_status dinr_train_path(dinr_ctx *c, int64_t n, int32_t *fused_kernel, int32_t *fused_dw_layers) {
  if (!c || !fused_kernel || !fused_dw_layers || n < 0) return DINR_EINVAL;
  if (!c->have_geom || !c->have_field) return fail(c, DINR_ESTATE, "geometry and field weights must be set first");
  Plan pl;
  plan_layout(c, std::max<int64_t>(n, 1), true, false, pl, nullptr);
  *fused_kernel = pl.fused ? (pl.fused2 ? 2 : 1) : 0;
  *fused_dw_layers = pl.fused ? pl.nf : 0;
  return DINR_OK;
}

dinr_status dinr_train_gemm_layers(dinr_ctx *c, int64_t n, int32_t *gl) {
  if (!c || !gl || n < 0) return c ? fail(c, DINR_EINVAL, "null array or n < 0") : DINR_EINVAL;
  if (!c->have_geom || !c->have_field) return fail(c, DINR_ESTATE, "geometry and field weights must be set first");
  Plan pl;
  plan_layout(c, std::max<int64_t>(n, 1), true, false, pl, nullptr);
  const int L = c->L;
  for (int k = 0; k < T_N; ++k) gl[k] = 0;
  if (c->field.precision == DINR_FP32_VERIFY) {  // SIMT verify path: forward, backward (dX + dW)
    gl[T_FWD] = L;
    gl[T_BWD] = (L - 1) + L;
  } else if (pl.fused) {
    // one fused kernel: forward, the dX chain down to layer lmin + 1, the TMEM-fused dW of the top
    // nf layers; k_dw01 (dw01): dW of layers 0 and 1 plus layer 1's dX (its layer-0 forward is a
    // recompute); otherwise K5: dW of the nu lower layers
    const int lmin = pl.dw01 ? 1 : 0;
    gl[T_BWD] = L + (L - 1 - lmin) + pl.nf;
    gl[T_DW] = pl.nu + lmin;
  } else {  // split path: K2 forward, K3 dX chain, K5 dW
    gl[T_FWD] = L;
    gl[T_BWD] = L - 1;
    gl[T_DW] = L;
  }
  return DINR_OK;
}

}  // extern "C"

// ------------------------------------------------------------------------------------------------
// N4 inference voxelization
namespace {

VoxGrid vox_grid(const dinr_ctx *c, const dinr_voxel_grid &g, double t, int64_t k0) {
  const dinr_geometry &ge = c->geom;
  VoxGrid v;
  v.nx = g.nx;
  v.ny = g.ny;
  v.k0 = k0;
  v.x0 = g.x0;
  v.y0 = g.y0;
  v.z0 = g.z0;
  v.vx = g.vx;
  v.vy = g.vy;
  v.vz = g.vz;
  v.xs0 = ge.rot_center_x;
  v.r = ge.fov_radius;
  v.zc = 0.5 * (ge.z_lo + ge.z_hi);
  v.zh = 0.5 * (ge.z_hi - ge.z_lo);
  const double tc = 0.5 * (ge.t_lo + ge.t_hi), th = 0.5 * (ge.t_hi - ge.t_lo);
  v.tbar = th > 0.0 ? (float)((t - tc) / th) : 0.f;
  return v;
}

template <int H>
bool infer_fits(const dinr_ctx *c) {
  return InferLayout<H>::smem_bytes(c->L) <= 227 * 1024;
}

template <int H>
dinr_status launch_infer(dinr_ctx *c, const VoxGrid &vg, int64_t n_vox, float *out, cudaStream_t st) {
  if (c->field.precision == DINR_BF16 && H <= 128 && infer_fits<H>(c)) {
    InferParams p{};
    p.vg = vg;
    p.n_vox = n_vox;
    p.L = c->L;
    p.mu0 = (float)c->field.mu0;
    p.params = c->d_params;
    p.B = c->d_B;
    p.wpack_half = c->d_wpack_half;
    p.out = out;
    const size_t smem = InferLayout<H>::smem_bytes(c->L);
    dinr_status s = set_smem(c, k_infer<H>, smem);
    if (s) return s;
    const int64_t groups = (n_vox + 255) / 256;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(groups, c->sm_count));
    Launch L_(c, T_FWD, st);
    k_infer<H><<<grid, InferLayout<H>::NT, smem, st>>>(p);
    CUDA_TRY(c, cudaGetLastError());
    return DINR_OK;
  }
  // general path (H = 256 or layers that do not fit): K2 in grid mode, weights streamed
  TcParams p{};
  p.nsamp = n_vox;
  p.n_s = 1;
  p.L = c->L;
  p.resident = tc_resident(H, c->L) ? 1 : 0;
  p.mu0 = (float)c->field.mu0;
  p.params = c->d_params;
  p.B = c->d_B;
  p.wpack = c->d_wpack;
  p.grid_mode = 1;
  p.vg = vg;
  p.vout = out;
  const size_t smem = TcLayout<H>::smem_bytes(c->L, p.resident != 0);
  dinr_status s = set_smem(c, k_tc_mlp<H, 0>, smem);
  if (s) return s;
  const int64_t tiles = (n_vox + 127) / 128;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)c->sm_count * tc_occupancy(c)));
  Launch L_(c, T_FWD, st);
  k_tc_mlp<H, 0><<<grid, kTcThreads, smem, st>>>(p);
  CUDA_TRY(c, cudaGetLastError());
  return DINR_OK;
}

dinr_status simt_voxelize(dinr_ctx *c, const VoxGrid &vg, int64_t n_vox, float *out, cudaStream_t st) {
  const int H = c->H, L = c->L;
  const int64_t per_pix = (int64_t)c->S * c->geom.samples_per_ray;
  Plan pl;
  dinr_status s = ensure_plan(c, (n_vox + per_pix - 1) / per_pix, false, false, pl);
  if (s) return s;
  {
    Launch L_(c, T_FWD, st);
    s_vox_features<<<(unsigned)((n_vox + 255) / 256), 256, 0, st>>>(vg, n_vox, c->d_B, c->C, pl.sh);
  }
  CUDA_TRY(c, cudaGetLastError());
  const int64_t per = (int64_t)H * H + H;
  for (int l = 0; l < L; ++l) {
    SgemmArgs a{};
    a.A = pl.sh + (size_t)l * n_vox * H;
    a.sam = H;
    a.sak = 1;
    a.B = c->d_params + l * per;
    a.sbk = 1;
    a.sbn = H;
    a.M = n_vox;
    a.N = H;
    a.K = H;
    a.kchunk = H;
    a.mode = 1;
    a.ldc = H;
    a.bias = c->d_params + l * per + (int64_t)H * H;
    a.Z = pl.sz + (size_t)l * n_vox * H;
    a.Hout = pl.sh + (size_t)(l + 1) * n_vox * H;
    s = simt_gemm(c, a, 1, st, T_FWD);
    if (s) return s;
  }
  {
    Launch L_(c, T_FWD, st);
    s_vox_head<<<(unsigned)((n_vox + 255) / 256), 256, 0, st>>>(vg, pl.sh + (size_t)L * n_vox * H, n_vox, H,
                                                              c->d_params + L * per, (float)c->field.mu0, out);
  }
  CUDA_TRY(c, cudaGetLastError());
  return DINR_OK;
}

dinr_status voxelize_slab(dinr_ctx *c, const dinr_voxel_grid &g, double t, int64_t k0, int64_t kn, float *out,
                          cudaStream_t st) {
  const VoxGrid vg = vox_grid(c, g, t, k0);
  const int64_t n_vox = g.nx * g.ny * kn;
  if (c->field.precision == DINR_FP32_VERIFY) return simt_voxelize(c, vg, n_vox, out, st);
  switch (c->H) {
    case 64: return launch_infer<64>(c, vg, n_vox, out, st);
    case 128: return launch_infer<128>(c, vg, n_vox, out, st);
    default: return launch_infer<256>(c, vg, n_vox, out, st);
  }
}

bool grid_ok(const dinr_voxel_grid *g) {
  return g && g->nx > 0 && g->ny > 0 && g->nz > 0 && g->vx > 0 && g->vy > 0 && g->vz > 0 &&
         std::isfinite(g->x0) && std::isfinite(g->y0) && std::isfinite(g->z0) && g->nx * g->ny <= (int64_t)1 << 40;
}

}  // namespace

extern "C" {

dinr_status dinr_default_grid(dinr_ctx *c, dinr_voxel_grid *out) {
  if (!c || !out) return DINR_EINVAL;
  if (!c->have_geom) return fail(c, DINR_ESTATE, "geometry must be set first");
  const dinr_geometry &g = c->geom;
  const double mag = g.beam == DINR_PARALLEL ? 1.0 : (g.sod + g.odd) / g.sod;
  const double vx = g.pixel_dx / mag, vz = g.pixel_dz / mag, r = g.fov_radius;
  out->vx = out->vy = vx;
  out->vz = vz;
  out->nx = out->ny = (int64_t)std::ceil(2.0 * r / vx);
  out->nz = std::max<int64_t>(1, (int64_t)std::ceil((g.z_hi - g.z_lo) / vz));
  out->x0 = g.rot_center_x - 0.5 * (double)out->nx * vx;
  out->y0 = -0.5 * (double)out->ny * vx;
  out->z0 = 0.5 * (g.z_lo + g.z_hi) - 0.5 * (double)out->nz * vz;
  return DINR_OK;
}

dinr_status dinr_voxelize(dinr_ctx *c, const dinr_voxel_grid *g, double t, int64_t k_begin, int64_t k_count,
                          float *out_dev, void *stream) {
  if (!c) return DINR_EINVAL;
  if (!c->have_geom || !c->have_field) return fail(c, DINR_ESTATE, "geometry and field weights must be set first");
  if (!grid_ok(g) || !out_dev || k_begin < 0 || k_count <= 0 || k_begin + k_count > g->nz || !std::isfinite(t))
    return fail(c, DINR_EINVAL, "bad voxel grid or slab");
  CUDA_TRY(c, cudaSetDevice(c->device));
  return voxelize_slab(c, *g, t, k_begin, k_count, out_dev, (cudaStream_t)stream);
}

dinr_status dinr_voxelize_to_file(dinr_ctx *c, const dinr_voxel_grid *g, int64_t view_begin, int64_t n_views,
                                  const char *path, int64_t slab_planes) {
  if (!c) return DINR_EINVAL;
  if (!c->have_geom || !c->have_field) return fail(c, DINR_ESTATE, "geometry and field weights must be set first");
  if (!grid_ok(g) || !path || view_begin < 0 || n_views < 0 || view_begin + n_views > c->M || slab_planes <= 0)
    return fail(c, DINR_EINVAL, "bad voxel grid, view range or slab size");
  CUDA_TRY(c, cudaSetDevice(c->device));
  FILE *fh = std::fopen(path, "wb");
  if (!fh) return fail(c, DINR_ECUDA, std::string("cannot open ") + path);
  const int64_t kp = std::min(slab_planes, g->nz);
  const size_t slab = (size_t)(g->nx * g->ny * kp);
  float *dbuf[2] = {nullptr, nullptr}, *hbuf[2] = {nullptr, nullptr};
  cudaStream_t st = nullptr;
  cudaEvent_t done[2] = {nullptr, nullptr};
  dinr_status rs = DINR_OK;
  auto cleanup = [&]() {
    if (st) cudaStreamSynchronize(st);
    for (int b = 0; b < 2; ++b) {
      cudaFree(dbuf[b]);
      cudaFreeHost(hbuf[b]);
      if (done[b]) cudaEventDestroy(done[b]);
    }
    if (st) cudaStreamDestroy(st);
    std::fclose(fh);
  };
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
    cleanup();
    return fail(c, DINR_ECUDA, "stream creation failed");
  }
  for (int b = 0; b < 2; ++b)
    if (cudaMalloc(&dbuf[b], slab * sizeof(float)) != cudaSuccess ||
        cudaMallocHost(&hbuf[b], slab * sizeof(float)) != cudaSuccess ||
        cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming) != cudaSuccess) {
      cleanup();
      return fail(c, DINR_ENOMEM, "voxel slab buffers");
    }
  // slab q: compute into dbuf[q%2], copy to hbuf[q%2], record done[q%2]; the host writes slab q-1
  // while slab q is on the GPU
  int64_t pending = -1, pending_n = 0;
  int64_t q = 0;
  for (int64_t m = view_begin; m < view_begin + n_views && rs == DINR_OK; ++m)
    for (int64_t k0 = 0; k0 < g->nz && rs == DINR_OK; k0 += kp, ++q) {
      const int64_t kn = std::min(kp, g->nz - k0);
      const int b = (int)(q & 1);
      if (pending >= 0 && (pending & 1) == b) {  // both buffers busy: drain the older one first
        cudaEventSynchronize(done[b]);
        if (std::fwrite(hbuf[b], sizeof(float), (size_t)pending_n, fh) != (size_t)pending_n)
          rs = fail(c, DINR_ECUDA, std::string("write failed: ") + path);
        pending = -1;
      }
      if (rs) break;
      rs = voxelize_slab(c, *g, c->h_t[m], k0, kn, dbuf[b], st);
      if (rs) break;
      const int64_t n = g->nx * g->ny * kn;
      if (cudaMemcpyAsync(hbuf[b], dbuf[b], (size_t)n * sizeof(float), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
          cudaEventRecord(done[b], st) != cudaSuccess) {
        rs = fail(c, DINR_ECUDA, "slab copy failed");
        break;
      }
      if (pending >= 0) {  // write the previous slab while this one computes
        const int pb = (int)(pending & 1);
        cudaEventSynchronize(done[pb]);
        if (std::fwrite(hbuf[pb], sizeof(float), (size_t)pending_n, fh) != (size_t)pending_n)
          rs = fail(c, DINR_ECUDA, std::string("write failed: ") + path);
      }
      pending = q;
      pending_n = n;
    }
  if (rs == DINR_OK && pending >= 0) {
    const int pb = (int)(pending & 1);
    if (cudaEventSynchronize(done[pb]) != cudaSuccess)
      rs = fail(c, DINR_ECUDA, "slab compute failed");
    else if (std::fwrite(hbuf[pb], sizeof(float), (size_t)pending_n, fh) != (size_t)pending_n)
      rs = fail(c, DINR_ECUDA, std::string("write failed: ") + path);
  }
  cleanup();
  return rs;
}

}  // extern "C"
