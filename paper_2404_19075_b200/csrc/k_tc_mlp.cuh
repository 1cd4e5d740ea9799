// k_tc_mlp.cuh -- K2 (fused sample -> GRFF -> L x (tcgen05 GEMM + bias + Swish) -> head ->
// ray-chunk sum) and K3 (same forward recomputed, then the backward dX chain on the tensor
// cores), north_star subsystems (2) and (3).
//
// Tile = 128 consecutive samples (rows) = 128 TMEM lanes; one CTA of 128 threads, thread r
// owns row r (its sample) in every epilogue; thread 0 issues the tcgen05.mma and the bulk
// (TMA-engine) copies.  Per layer l the accumulator D[128 x H] (fp32, TMEM) is
//   forward : D = A(h_l, K-major SW128 smem) . W_l^T   (B = W_l image, K-major)
//   backward: D = A(delta_l)                  . W_l     (B = same W_l image, MN-major)
// Weights live in shared memory for the whole kernel when L*H*H*2 fits (H <= 128), else they
// are streamed one layer at a time with a prefetch issued as soon as the previous MMA retires.
// K3 writes, per tile, the bf16 images of h_l (layer inputs) and delta_l with bulk
// shared->global copies (operands of the dW GEMM, k_tc_dw.cuh), keeps z_l in an fp16
// coalesced stash for swish', and reduces the head gradients (dL/dw_o = sum u h_L,
// dL/db_o = sum u) with a warp transpose-reduction into registers.
#pragma once
#include "internal.cuh"
#include "k_features.cuh"
#include "ptx_sm100.cuh"

namespace dinr {

struct TcParams {
  const float4 *rec32;
  Jitter jit;  // N3 sample placement
  int64_t nsamp;
  int n_s;
  int L;
  int resident;
  float mu0;
  const float *params;
  const float *B;
  const uint16_t *wpack;
  float *pchunk;   // forward: [nsamp/32] sums of M over 32-sample chunks
  // training
  const float *u;  // [n_rays] upstream for the raw head output (K4)
  uint8_t *hstash, *dstash, *zstash;
  float *head_part;  // [gridDim.x][H+1]
  int64_t n_tiles;
  int stash_feat;  // MODE 1: store layer 0's input tile (0: the dW GEMM recomputes the features)
  // N4 inference: samples are voxel centres of vg, outputs per voxel to vout (forward only)
  int grid_mode;
  VoxGrid vg;
  float *vout;
  unsigned long long *dbg;  // DINR_PHASES builds: per-CTA cycle counters (k_tc_fwd3)
  // H = 256 split path with k_tc_fwd3: the forward stashes only y_l = z_l / 2 (fp16, every layer;
  // no h stash, no swish' stash); K3 recomputes swish'(z) and the dW GEMM recomputes h = swish(z)
  int zall;
  float *db3;  // zall: per-CTA bias-gradient partials [L][2 m-blocks][gridDim.x][128] (K3's ones-MMA)
};

template <int H>
struct TcLayout {
  static constexpr uint32_t A_BYTES = H * 256u;        // 128 rows x H bf16
  static constexpr uint32_t W_LAYER = H * H * 2u;
  static size_t smem_bytes(int L, bool resident) {
    size_t w = resident ? (size_t)L * W_LAYER : W_LAYER;
    return 1024 + A_BYTES + w + 2048 + (size_t)L * H * 4 + H * 4 + 16 + (H / 2) * 16 + 64 + 2 * 128 * 4;
  }
};

// ray of sample g: 32-bit division whenever g fits (every training batch; the 64-bit division is
// a long subroutine call)
__device__ __forceinline__ int64_t ray_of(int64_t g, int n_s) {
  return (g >> 32) == 0 ? (int64_t)((uint32_t)g / (uint32_t)n_s) : g / n_s;
}

__device__ __forceinline__ float swish_f(float z) { return z * (0.5f + 0.5f * tanh_approx(0.5f * z)); }
__device__ __forceinline__ float dswish_f(float z) {
  float s = 0.5f + 0.5f * tanh_approx(0.5f * z);
  return s * (1.f + z * (1.f - s));
}

// 256 threads: thread = (TMEM lane / sample row, column half cg); every MMA is issued as two
// N = H/2 halves with their own commit, so half cg's epilogue starts while the other half computes.
constexpr int kTcThreads = 256;

// MODE 0: forward (projection / voxels: ray-chunk sums or per-voxel values)
// MODE 1: training forward: as 0, plus bulk stores of every layer input h_l and fp16 z_l stores
// MODE 2: training backward from the stashes: top-layer delta and head gradients from z_{L-1},
//         then the dX chain (K3); no forward recompute
// MODE 3: MODE 2 on the y-only stash of k_tc_fwd3 (H = 256, DINR_ZALL): swish' recomputed from
//         y = z / 2, and db accumulated by a ones-MMA (the dW GEMM k_tc_dwz has no TMEM for it)
template <int H, int MODE>
__global__ void __launch_bounds__(kTcThreads, 1) k_tc_mlp(TcParams p) {
  constexpr bool TRAIN = MODE == 2 || MODE == 3;
  constexpr bool ZALL = MODE == 3;  // MODE 3: MODE 2 on the y-only stash (k_tc_fwd3 zall), H = 256
  constexpr int C = H / 2;
  constexpr uint32_t A_BYTES = TcLayout<H>::A_BYTES;
  constexpr uint32_t W_LAYER = TcLayout<H>::W_LAYER;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared address space
  const int L = p.L;
  const bool resident = p.resident != 0;
  uint8_t *sA = smem;
  uint8_t *sW = smem + A_BYTES;
  uint8_t *sOnes = sW + (resident ? (size_t)L * W_LAYER : (size_t)W_LAYER);  // K3 zall: bf16 ones (db MMA)
  float *sBias = reinterpret_cast<float *>(sOnes + 2048);
  float *sWo = sBias + L * H;
  float *sB = sWo + H + 4;
  uint64_t *bars = reinterpret_cast<uint64_t *>(sB + C * 4);
  uint64_t *mma_bar = bars, *w_bar = bars + 2;  // mma_bar[cg]: N-half cg of the current MMA retired
  uint64_t *sa_ok = bars + 3;                    // MODE 1: sA may be rewritten (see the epilogue)
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 4);
  uint64_t *db_bar = bars + 5;
  uint64_t *w_bar1 = bars + 6;  // K3 at H = 256: second half of the streamed W_l (sMu starts after it)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // K3 on the zall path also accumulates db_l = sum_samples delta_l with a ones-MMA per m-block
  // into TMEM columns [H, H + 2L 16) for the CTA's life (the dW GEMM then has no room for it)
  constexpr bool dbm = ZALL && H == 256;
  const uint32_t tcols = dbm ? 512u : (uint32_t)H;
  if (warp == 0) {
    tmem_alloc(tmem_slot, tcols);
    tmem_relinquish();
  }
  if (tid == 0) {
    mbar_init(&mma_bar[0], 1);
    mbar_init(&mma_bar[1], 1);
    mbar_init(w_bar, 1);
    mbar_init(sa_ok, 1);
    mbar_init(db_bar, 1);
    mbar_init(w_bar1, 1);
    fence_mbar_init();
  }
  if (dbm) {
    for (int i = tid; i < 2048 / 4; i += kTcThreads) reinterpret_cast<uint32_t *>(sOnes)[i] = 0x3F803F80u;
    fence_proxy_async_smem();
  }
  const int64_t per = (int64_t)H * H + H;
  for (int i = tid; i < L * H; i += kTcThreads) sBias[i] = p.params[(i / H) * per + (int64_t)H * H + (i % H)];
  for (int i = tid; i <= H; i += kTcThreads) sWo[i] = p.params[(int64_t)L * per + i];  // w_o, then b_o
  for (int i = tid; i < C * 4; i += kTcThreads) sB[i] = p.B[i];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t a_base = smem_u32(sA), w_base = smem_u32(sW);
  const uint32_t tmem_row = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  const int cg = tid >> 7;                     // column half of this thread
  const int cb_lo = cg * (H / 64);  // first of its H/64 32-column chunks
  float *sMu = reinterpret_cast<float *>(bars + 7);  // [2][128] per-half head partials (forward)
  // the training plan may round the tile count up (paired tiles): padding tiles hold invalid samples
  const int n_tiles = (int)(p.n_tiles > (p.nsamp + 127) / 128 ? p.n_tiles : (p.nsamp + 127) / 128);

  // Weight schedule (thread 0): the layer whose image sits in sW, and a pending load.
  int w_cur = -1;
  uint32_t w_phase = 0;
  bool w_pending = false;
  auto w_issue = [&](int layer) {  // only when no MMA is reading sW
    uint32_t bytes = resident ? (uint32_t)L * W_LAYER : W_LAYER;
    const uint8_t *src = reinterpret_cast<const uint8_t *>(p.wpack) + (resident ? 0 : (size_t)layer * W_LAYER);
    mbar_arrive_expect_tx(w_bar, bytes);
    for (uint32_t off = 0; off < bytes; off += 32768u)
      bulk_g2s(sW + off, src + off, min(32768u, bytes - off), w_bar);
    w_pending = true;
    w_cur = resident ? -2 : layer;
  };
  auto w_ready = [&](int layer) -> uint32_t {
    if (w_pending) {
      mbar_wait(w_bar, w_phase);
      w_phase ^= 1;
      w_pending = false;
    }
    return resident ? w_base + (uint32_t)layer * W_LAYER : w_base;
  };
  // K3 streaming H = 256: W_l in two 64 KB halves (the MN-major blocks of input features [128 h,
  // +128), one per dX MMA half) with their own barriers, so the next layer's half h loads as soon as
  // this layer's half-h MMA has retired and the next half-0 MMA waits for 64 KB, not 128
  constexpr bool kHalfW = TRAIN && H == 256;
  uint32_t wh_phase[2] = {0, 0};
  bool wh_pending[2] = {false, false};
  uint64_t *wh_bar[2] = {w_bar, w_bar1};
  auto wh_issue = [&](int layer, int h) {
    mbar_arrive_expect_tx(wh_bar[h], W_LAYER / 2);
    const uint8_t *src = reinterpret_cast<const uint8_t *>(p.wpack) + (size_t)layer * W_LAYER + (size_t)h * (W_LAYER / 2);
    bulk_g2s(sW + h * (W_LAYER / 2), src, W_LAYER / 4, wh_bar[h]);
    bulk_g2s(sW + h * (W_LAYER / 2) + W_LAYER / 4, src + W_LAYER / 4, W_LAYER / 4, wh_bar[h]);
    wh_pending[h] = true;
  };
  auto wh_ready = [&](int h) {
    if (wh_pending[h]) {
      mbar_wait(wh_bar[h], wh_phase[h]);
      wh_phase[h] ^= 1;
      wh_pending[h] = false;
    }
  };
  if (tid == 0 && (int)blockIdx.x < n_tiles && (!TRAIN || L >= 2)) {
    if (kHalfW && !resident) {
      wh_issue(L - 1, 0);
      wh_issue(L - 1, 1);
    } else {
      w_issue(TRAIN ? L - 1 : 0);
    }
  }

  uint32_t mma_phase = 0, sa_phase = 0;
  constexpr int NCB = H / 64;  // 32-column chunks of this thread's column half
  float head_acc[NCB];
#pragma unroll
  for (int i = 0; i < NCB; ++i) head_acc[i] = 0.f;
  float bo_acc = 0.f;
  const uint64_t pol_z = policy_evict_first();  // z stash: written once, read once by the next kernel
  constexpr bool kSplit = H >= 128;  // N halves need whole 64-column blocks for the MN-major dX operand
  constexpr int NH = kSplit ? H / 2 : H;
  const uint32_t idesc_f = idesc_bf16(128, NH, 0, 0);
  const uint32_t idesc_b = idesc_bf16(128, NH, 0, 1);

  bool db_first = true;  // the CTA's first tile: the db accumulators start fresh
  uint32_t db_phase = 0;
  const uint32_t ones_a = smem_u32(sOnes);
  const uint32_t idesc_db = idesc_bf16(128, 16, 1, 0);  // A = delta^T (MN-major), B = ones (K-major)
  auto issue_db = [&](int l) {  // thread 0: db_l += sum over the tile's samples of delta_l, per m-block
    tc_fence_after();
#pragma unroll
    for (int mb = 0; mb < 2; ++mb)
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        umma_bf16(tmem + H + (uint32_t)(l * 2 + mb) * 16, sdesc_sw128(a_base + mb * 32768 + kk * 2048, 16384, 1024),
                  sdesc_sw128(ones_a + (kk & 3) * 32, 16, 1024), idesc_db, (!db_first || kk > 0) ? 1u : 0u);
  };
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const bool more_tiles = tile + (int)gridDim.x < n_tiles;
    const int row = tid & 127;
    const int64_t g = (int64_t)tile * 128 + row;
    const bool valid = g < p.nsamp;
    bool inside = false;
    if (TRAIN) {  // the previous tile's last bulk store must be done reading sA
      if (tid == 0) bulk_wait_read_all();
      __syncthreads();
    }
    if (!TRAIN) {
      // ---------------------------------------------------------------- a5/a6 features
      {
        float rb0 = 0.f, rb1 = 0.f, rb2 = 0.f, rb3 = 0.f;
        if (MODE == 0 && p.grid_mode) {
          const float4 r = voxel_coords(p.vg, valid ? g : 0, inside);
          rb0 = r.x;
          rb1 = r.y;
          rb2 = r.z;
          rb3 = r.w;
        } else if (valid) {
          int64_t ray = ray_of(g, p.n_s);
          const uint32_t jr = (uint32_t)(g - ray * p.n_s);
          float jj = (float)jr + sample_offset(p.jit, ray, jr);
          float4 ra = p.rec32[2 * ray], rbv = p.rec32[2 * ray + 1];
          rb0 = ra.w;                 // t
          rb1 = ra.z + jj * rbv.z;    // z
          rb2 = ra.y + jj * rbv.y;    // y
          rb3 = ra.x + jj * rbv.x;    // x
        }
#pragma unroll 1
        for (int c0 = cg * (C / 2); c0 < (cg + 1) * (C / 2); c0 += 16) {
          uint32_t pc[8], ps[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            float cs[2], sn[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const float *bb = sB + 4 * (c0 + 2 * q + e);
              float phi = bb[0] * rb0 + bb[1] * rb1 + bb[2] * rb2 + bb[3] * rb3;
              float fr = phi - rintf(phi);  // range reduction to [-1/2, 1/2]
              __sincosf(6.283185307179586f * fr, &sn[e], &cs[e]);
            }
            pc[q] = pack_bf16x2(cs[0], cs[1]);
            ps[q] = pack_bf16x2(sn[0], sn[1]);
          }
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            st_shared_v4(a_base + sw128_offset(row, c0 + 8 * hh, 128), pc[4 * hh], pc[4 * hh + 1], pc[4 * hh + 2], pc[4 * hh + 3]);
            st_shared_v4(a_base + sw128_offset(row, C + c0 + 8 * hh, 128), ps[4 * hh], ps[4 * hh + 1], ps[4 * hh + 2],
                         ps[4 * hh + 3]);
          }
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncthreads();
      if (MODE == 1 && p.stash_feat && tid == 0) {  // layer 0's input for the dW GEMM (unless it recomputes it)
        bulk_s2g(p.hstash + ((size_t)0 * p.n_tiles + tile) * A_BYTES, sA, A_BYTES);
        bulk_commit();
      }
      // ---------------------------------------------------------------- a7/a8 forward
      float mu_acc = 0.f;
      for (int l = 0; l < L; ++l) {
        if (tid == 0) {
          uint32_t wl = w_ready(l);
          tc_fence_after();
          for (int half = 0; half < 2; ++half) {  // output columns [half NH, (half+1) NH)
            if (half == 0 || kSplit) {
#pragma unroll 4
              for (int kk = 0; kk < H / 16; ++kk) {
                uint64_t ad = sdesc_sw128(a_base + (kk >> 2) * (128 * 128) + (kk & 3) * 32, 16, 1024);
                uint64_t bd = sdesc_sw128(wl + (kk >> 2) * (H * 128) + half * NH * 128 + (kk & 3) * 32, 16, 1024);
                umma_bf16(tmem + half * NH, ad, bd, idesc_f, kk > 0 ? 1u : 0u);
              }
            }
            umma_commit(&mma_bar[half]);
          }
        }
        mbar_wait(&mma_bar[cg], mma_phase);
        mma_phase ^= 1;
        tc_fence_after();
        const bool last = (l == L - 1);
        // this thread's half of the layer output, kept in registers until the other half's MMA
        // (which reads all of sA) has retired: h_{l+1} overwrites sA in place
        uint32_t hk[NCB][16];
#pragma unroll
        for (int c = 0; c < NCB; ++c) {
          const int cb = cb_lo + c;
          uint32_t v[32];
          tmem_ld32(tmem_row + cb * 32, v);
          tmem_wait_ld();
          float z[32], sg[32];  // pre-activation and its sigmoid (one tanh per element)
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            z[i] = __uint_as_float(v[i]) + sBias[l * H + cb * 32 + i];
            sg[i] = 0.5f + 0.5f * tanh_approx(0.5f * z[i]);
          }
          if (MODE == 1) {  // backward state, [16-column chunk][row][32 B]: swish'(z_l) as bf16 for the
                            // hidden layers (no tanh in the backward), z_{L-1} as fp16 for the top layer
#pragma unroll
            for (int qq = 0; qq < 2; ++qq) {
              uint32_t h8[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const int i0 = 16 * qq + 2 * e;
                if (last) {
                  __half2 hh = __floats2half2_rn(z[i0], z[i0 + 1]);
                  h8[e] = *reinterpret_cast<uint32_t *>(&hh);
                } else {  // swish'(z) = s (1 + z (1 - s))
                  h8[e] = pack_bf16x2(sg[i0] * (1.f + z[i0] * (1.f - sg[i0])),
                                      sg[i0 + 1] * (1.f + z[i0 + 1] * (1.f - sg[i0 + 1])));
                }
              }
              st_global_v8_hint(p.zstash + ((((size_t)l * p.n_tiles + tile) * (H / 16) + (cb * 2 + qq)) * 128 + row) * 32,
                                h8, pol_z);
            }
          }
          if (!last) {
#pragma unroll
            for (int i = 0; i < 16; ++i) hk[c][i] = pack_bf16x2(z[2 * i] * sg[2 * i], z[2 * i + 1] * sg[2 * i + 1]);  // swish = z s
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) mu_acc += sWo[cb * 32 + i] * (z[i] * sg[i]);
          }
        }
        if (MODE == 1) {
          // sA is rewritten below: both MMA halves and the bulk stash store of this layer's input
          // must be done reading it; thread 0 (which issued the store) publishes that on sa_ok
          if (tid == 0) {
            mbar_wait(&mma_bar[1], mma_phase ^ 1);
            bulk_wait_read_all();
            if (!last) mbar_arrive(sa_ok);
          } else if (!last) {
            mbar_wait(sa_ok, sa_phase);
          }
          if (!last) sa_phase ^= 1;
        } else if (cg == 0 && (!last || tid == 0)) {
          mbar_wait(&mma_bar[1], mma_phase ^ 1);  // both halves retired
        }
        if (tid == 0 && !resident) {  // prefetch the next weight image (streaming mode) now that sW is free
          const int nxt = (l + 1) % L;
          const bool has_next = (l + 1 < L) || more_tiles;
          if (has_next && nxt != w_cur) w_issue(nxt);
        }
        if (!last) {
#pragma unroll
          for (int c = 0; c < NCB; ++c)
#pragma unroll
            for (int q = 0; q < 4; ++q)
              st_shared_v4(a_base + sw128_offset(row, (cb_lo + c) * 32 + 8 * q, 128), hk[c][4 * q], hk[c][4 * q + 1],
                           hk[c][4 * q + 2], hk[c][4 * q + 3]);
          fence_proxy_async_smem();
        }
        tc_fence_before();
        __syncthreads();
        if (MODE == 1 && !last && tid == 0) {  // input of layer l+1 for the dW GEMM
          bulk_s2g(p.hstash + ((size_t)(l + 1) * p.n_tiles + tile) * A_BYTES, sA, A_BYTES);
          bulk_commit();
        }
      }
      // a9 ray-chunk sum of M = mu0 (w_o . h_L + b_o) over the warp's 32 samples (the two column
      // halves of a row meet in shared memory)
      sMu[cg * 128 + row] = mu_acc;
      __syncthreads();
      if (cg == 0) {
        float mu = p.mu0 * (sMu[row] + sMu[128 + row] + sWo[H]);
        if (MODE == 0 && p.grid_mode) {
          if (valid) p.vout[g] = inside ? mu : 0.f;
        } else {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) mu += __shfl_xor_sync(0xffffffffu, mu, o);
          if (lane == 0 && valid) p.pchunk[g >> 5] = mu;
        }
      }
    } else {
      // ---------------------------------------------------------------- a12 backward (MODE 2)
      // top layer from the stashed z_{L-1}: h_L = swish(z) for the head gradients (transpose-
      // reduce u h_L over the warp's 32 rows), delta_L = u w_o swish'(z)
      const float u_row = valid ? p.u[ray_of(g, p.n_s)] : 0.f;
      constexpr float zscale = ZALL ? 2.f : 1.f;
      constexpr uint32_t kZTile = 128u * H * 2u;  // one tile of fp16 z
      if (tid == 0 && L >= 2)  // z_{L-2} is read after the first dX: bring it to L2 now
        bulk_prefetch_l2(p.zstash + ((size_t)(L - 2) * p.n_tiles + tile) * kZTile, kZTile);
      {
        const uint8_t *zsrc = p.zstash + (((size_t)(L - 1) * p.n_tiles + tile) * (H / 16) * 128 + row) * 32;
        uint4 zt[NCB][4];  // all of this thread's z chunks in flight at once
#pragma unroll
        for (int c = 0; c < NCB; ++c)
#pragma unroll
          for (int qq = 0; qq < 2; ++qq)
            ld_global_v8_hint(zsrc + (size_t)((cb_lo + c) * 2 + qq) * 128 * 32, zt[c][2 * qq], zt[c][2 * qq + 1], pol_z);
#pragma unroll
        for (int c = 0; c < NCB; ++c) {
          const int cb = cb_lo + c;
          float z[32];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint4 zq = zt[c][q];
            const uint32_t zz[4] = {zq.x, zq.y, zq.z, zq.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 zf = __half22float2(*reinterpret_cast<const __half2 *>(&zz[e]));
              z[8 * q + 2 * e] = zscale * zf.x;  // zall: the stash holds y = z / 2 (exact scaling)
              z[8 * q + 2 * e + 1] = zscale * zf.y;
            }
          }
          float x[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) x[i] = u_row * swish_f(z[i]);
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) {
            const bool upper = (lane & o) != 0;
#pragma unroll
            for (int i = 0; i < o; ++i) {
              float send = upper ? x[i] : x[i + o];
              float keep = upper ? x[i + o] : x[i];
              x[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
          }
          head_acc[c] += x[0];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t w4[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              int i0 = 8 * q + 2 * e;
              float d0 = u_row * sWo[cb * 32 + i0] * dswish_f(z[i0]);
              float d1 = u_row * sWo[cb * 32 + i0 + 1] * dswish_f(z[i0 + 1]);
              w4[e] = pack_bf16x2(d0, d1);
            }
            st_shared_v4(a_base + sw128_offset(row, cb * 32 + 8 * q, 128), w4[0], w4[1], w4[2], w4[3]);
          }
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncthreads();
        if (tid == 0) {
          bulk_s2g(p.dstash + ((size_t)(L - 1) * p.n_tiles + tile) * A_BYTES, sA, A_BYTES);
          bulk_commit();
          if (dbm) issue_db(L - 1);
        }
      }
      if (cg == 0) {
        float us = u_row;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) us += __shfl_xor_sync(0xffffffffu, us, o);
        bo_acc += us;
      }
      // dX chain
      for (int l = L - 1; l >= 1; --l) {
        // swish'(z_{l-1}) of this thread's chunks: loads in flight while the dX MMA runs
        uint4 zq[NCB][4];
        {
          const uint8_t *zsrc = p.zstash + (((size_t)(l - 1) * p.n_tiles + tile) * (H / 16) * 128 + row) * 32;
#pragma unroll
          for (int c = 0; c < NCB; ++c)
#pragma unroll
            for (int qq = 0; qq < 2; ++qq)
              ld_global_v8_hint(zsrc + (size_t)((cb_lo + c) * 2 + qq) * 128 * 32, zq[c][2 * qq], zq[c][2 * qq + 1], pol_z);
        }
        if (tid == 0) {
          uint32_t wl = (kHalfW && !resident) ? w_base : w_ready(l);
          // z of the next step (or the next tile's top layer) into L2 while this step runs
          if (l >= 2)
            bulk_prefetch_l2(p.zstash + ((size_t)(l - 2) * p.n_tiles + tile) * kZTile, kZTile);
          else if (more_tiles)
            bulk_prefetch_l2(p.zstash + ((size_t)(L - 1) * p.n_tiles + tile + gridDim.x) * kZTile, kZTile);
          for (int half = 0; half < 2; ++half) {  // input columns [half NH, (half+1) NH)
            if (kHalfW && !resident) wh_ready(half);
            tc_fence_after();
            if (half == 0 || kSplit) {
#pragma unroll 4
              for (int kk = 0; kk < H / 16; ++kk) {
                uint64_t ad = sdesc_sw128(a_base + (kk >> 2) * (128 * 128) + (kk & 3) * 32, 16, 1024);
                uint64_t bd = sdesc_sw128(wl + half * (NH / 64) * (H * 128) + kk * 2048, H * 128, 1024);  // MN-major W_l
                umma_bf16(tmem + half * NH, ad, bd, idesc_b, kk > 0 ? 1u : 0u);
              }
            }
            umma_commit(&mma_bar[half]);
          }
        }
        mbar_wait(&mma_bar[cg], mma_phase);
        mma_phase ^= 1;
        tc_fence_after();
        if (tid == 0) {
          const int nxt = (l - 1 >= 1) ? l - 1 : L - 1;
          const bool has_next = (l - 1 >= 1) || more_tiles;
          if (kHalfW && !resident) {  // half 0 retired (waited above): reload it, then half 1
            if (has_next) wh_issue(nxt, 0);
            mbar_wait(&mma_bar[1], mma_phase ^ 1);
            if (has_next) wh_issue(nxt, 1);
          } else {
            mbar_wait(&mma_bar[1], mma_phase ^ 1);
            if (!resident) {  // next: layer l-1, or the next tile's top layer
              if (has_next && nxt != w_cur) w_issue(nxt);
            }
          }
          bulk_wait_read_all();
        }
        __syncthreads();
#pragma unroll
        for (int c = 0; c < NCB; ++c) {
          const int cb = cb_lo + c;
          uint32_t v[32];
          tmem_ld32(tmem_row + cb * 32, v);
          tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t zz[4] = {zq[c][q].x, zq[c][q].y, zq[c][q].z, zq[c][q].w};
            uint32_t w4[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {  // delta = e swish'(z), swish' stashed as bf16 by the forward
              int i0 = 8 * q + 2 * e;
              float s0, s1;
              if (ZALL) {  // swish'(z) from the stashed y = z / 2: s = (1 + tanh y) / 2, s (1 + 2 y (1 - s))
                const float2 yf = __half22float2(*reinterpret_cast<const __half2 *>(&zz[e]));
#ifdef DINR_ZALL_F32_TANH
                const float g0 = fmaf(0.5f, tanh_approx(yf.x), 0.5f), g1 = fmaf(0.5f, tanh_approx(yf.y), 0.5f);
#else  // bf16x2 tanh, one MUFU op for both: the same precision as the bf16 swish' stash of the default path
                const uint32_t tt = bf2_tanh(pack_bf16x2(yf.x, yf.y));
                const float g0 = fmaf(0.5f, bf16lo(tt), 0.5f), g1 = fmaf(0.5f, bf16hi(tt), 0.5f);
#endif
                s0 = fmaf(g0, 2.f * yf.x * (1.f - g0), g0);
                s1 = fmaf(g1, 2.f * yf.y * (1.f - g1), g1);
              } else {
                s0 = bf16lo(zz[e]);
                s1 = bf16hi(zz[e]);
              }
              w4[e] = pack_bf16x2(__uint_as_float(v[i0]) * s0, __uint_as_float(v[i0 + 1]) * s1);
            }
            st_shared_v4(a_base + sw128_offset(row, cb * 32 + 8 * q, 128), w4[0], w4[1], w4[2], w4[3]);
          }
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncthreads();
        if (tid == 0) {
          bulk_s2g(p.dstash + ((size_t)(l - 1) * p.n_tiles + tile) * A_BYTES, sA, A_BYTES);
          bulk_commit();
          if (dbm) issue_db(l - 1);
        }
      }
      if (dbm && tid == 0) {  // delta_0's db MMAs must retire before the next tile rewrites sA
        umma_commit(db_bar);
        mbar_wait(db_bar, db_phase);
        db_phase ^= 1;
      }
      db_first = false;
    }
  }
  if (TRAIN) {
    // thread 0 waited for the last db MMAs (db_bar): order the other warps' TMEM reads after it
    tc_fence_before();
    __syncthreads();
    if (dbm && warp < 4) {  // db partials: TMEM lane o = output feature o of m-block mb
      tc_fence_after();
      for (int l = 0; l < L; ++l)
#pragma unroll
        for (int mb = 0; mb < 2; ++mb) {
          uint32_t v[16];
          tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + H + (uint32_t)(l * 2 + mb) * 16, v);
          tmem_wait_ld();
          p.db3[(((size_t)l * 2 + mb) * gridDim.x + blockIdx.x) * 128 + warp * 32 + lane] =
              db_first ? 0.f : __uint_as_float(v[0]);
        }
    }
    // per-CTA head partials: [H] = dL/dw_o, [H] slot = dL/db_o; combine the 4 warps via smem
    __syncthreads();
    float *red = reinterpret_cast<float *>(sA);  // A tile is free now (all bulk reads waited below)
    if (tid == 0) bulk_wait_read_all();
    __syncthreads();
#pragma unroll
    for (int c = 0; c < NCB; ++c) red[warp * (H + 1) + (cb_lo + c) * 32 + lane] = head_acc[c];
    if (lane == 0) red[warp * (H + 1) + H] = bo_acc;  // (zero for column-half-1 warps)
    __syncthreads();
    for (int k = tid; k <= H; k += kTcThreads) {
      float acc = 0.f;
      const int w0 = (k < H && k >= H / 2) ? 4 : 0;  // the 4 warps of the column half holding k
      for (int w = w0; w < w0 + 4; ++w) acc += red[w * (H + 1) + k];
      p.head_part[(size_t)blockIdx.x * (H + 1) + k] = acc;
    }
    if (tid == 0) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, tcols);
  }
}

}  // namespace dinr
