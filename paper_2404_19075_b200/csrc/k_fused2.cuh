// k_fused2.cuh -- fused training step, two concurrent tile streams (v3 of the fused path).
//
// Same math and the same pixel-group contract as k_fused (256 % (S*N_s) == 0, H <= 128), but
// the two 128-sample tiles of a group run concurrently on two epilogue warpgroups, so the
// tensor core computes one tile's layer while the other tile's epilogue runs:
//   WG s (s = 0, 1; 8 warps, 256 threads) owns tile 2g+s; thread = TMEM lane / sample row r and
//   the H/2 columns of its column half; warp 16 lane 0 issues every tcgen05.mma / bulk copy,
//   serving the streams in order (s = 0 then 1) at every layer.
// TMEM: acc[s] = [s*H, (s+1)*H); dW of the top nf = min(L, 512/H - 2) layers at 2H + j*H.
// SMEM: W_1..W_{L-1} resident; one buffer XB holds W_0 during the forward phase (only the
// forward needs W_0: there is no e_{-1}) and the h_l reload for the fused dW MMAs during the
// backward phase; A_0, A_1 operand tiles.
// Per-tile state (s2 = 2 swish'(z) of every layer, h of the fused layers) goes through the
// per-CTA L2 ring (evict_last), h/delta images of the unfused layers to the dW GEMM stash.
#pragma once
#include "internal.cuh"
#include "k_features.cuh"
#include "k_fused.cuh"
#include "ptx_sm100.cuh"

namespace dinr {

#ifndef DINR_F2_SUSPEND_NS
#define DINR_F2_SUSPEND_NS 0
#endif
// epilogue-side waits: suspended try_wait (0 ns hint = plain spinning probe)
__device__ __forceinline__ void f2_wait(uint64_t *bar, uint32_t parity) {
  if (DINR_F2_SUSPEND_NS > 0)
    mbar_wait_sleep(bar, parity, DINR_F2_SUSPEND_NS);
  else
    mbar_wait(bar, parity);
}
#ifndef DINR_F2_CTL_NS
#define DINR_F2_CTL_NS 1000
#endif
// waits of the MMA-issuer / copy warps: suspended try_wait (DINR_F2_CTL_SPIN: plain spinning)
__device__ __forceinline__ void f2_ctl_wait(uint64_t *bar, uint32_t parity) {
#ifdef DINR_F2_CTL_SPIN
  mbar_wait(bar, parity);
#else
  mbar_wait_sleep(bar, parity, DINR_F2_CTL_NS);
#endif
}
// operand-tile handoff after the writers' generic-proxy smem writes are fenced:
//   default: the stream's 8 warps meet at a named barrier, one thread arrives (one mbarrier event
//            per handoff: fewer wake-ups of the warps sleeping on mbarriers)
//   DINR_F2_WARP_ARRIVE: one arrival per warp
__device__ __forceinline__ void f2_arrive_tile(uint64_t *bar, int stream) {
#ifdef DINR_F2_WARP_ARRIVE
  (void)stream;
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
#else
  asm volatile("bar.sync %0, 256;" ::"r"(2 + stream) : "memory");
  if ((threadIdx.x & 255) == 0) mbar_arrive(bar);
#endif
}
#ifdef DINR_F2_WARP_ARRIVE
constexpr int kF2TileArrivals = 8;
#else
constexpr int kF2TileArrivals = 1;
#endif


template <int H>
struct Fused2Layout {
  static constexpr int EPI = 512;                 // 2 warpgroups x 8 warps
  static constexpr int NT = EPI + 64;             // + MMA warp + copy warp
  static constexpr uint32_t TILE = H * 256u;      // one 128-row bf16 tile image
  static constexpr uint32_t A_BYTES = H == 64 ? 2 * TILE : TILE;  // H = 64: zero pad block for M = 128 dW
  static constexpr uint32_t W_LAYER = H * H * 2u;
  static constexpr uint32_t XB = TILE > W_LAYER ? TILE : W_LAYER;
  static constexpr int NF_MAX = 512 / H - 2;
  static constexpr uint32_t ONES = 128 * 32;  // no-swizzle [128 rows][16] bf16: columns 0, 1 = 1
  static constexpr uint32_t BIAS_B = H * 32;  // no-swizzle [H rows][16] bf16: hi, lo of b_l / 2
  static size_t smem_bytes(int L) {
    return 1024 + 2 * (size_t)A_BYTES + XB + (size_t)(L - 1) * W_LAYER + ONES + (size_t)L * BIAS_B + (H + 4) * 4 +
           (H / 2) * 16 + 2 * 4 * (H + 4) * 4 + 3 * 64 * 4 + 256;
  }
};

template <int H>
__global__ void __launch_bounds__(Fused2Layout<H>::NT, 1) k_fused2(FusedParams p) {
  using LY = Fused2Layout<H>;
  constexpr int C = H / 2;
  constexpr int EPI = LY::EPI;
  constexpr int NCH = H / 64;  // 32-column chunks per thread (column half of H)
  constexpr uint32_t TILE = LY::TILE;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared address space
  const int L = p.L, nf = p.nf, nu = L - nf;  // unfused layers 0..nu-1 go through the dW GEMM
  // lowest backward step run here: with k_dw01, delta_0 = (delta_1 W_1) swish'(z_0) is formed there
  const int lmin = p.dw01 ? 1 : 0;
  uint8_t *sA0 = smem;
  uint8_t *sXB = sA0 + 2 * LY::A_BYTES;
  uint8_t *sW = sXB + LY::XB;  // W_1..W_{L-1}
  // biases enter the MMA as one extra K = 16 step: [1 1 0 ..] x [hi lo 0 ..]^T = b_l / 2 in fp32
  uint8_t *sOnes = sW + (size_t)(L - 1) * LY::W_LAYER;
  uint8_t *sBiasB = sOnes + LY::ONES;
  float *sWo = reinterpret_cast<float *>(sBiasB + (size_t)L * LY::BIAS_B);  // w_o[H], b_o
  float *sB = sWo + H + 4;                                                       // C x 4
  float *sHsum = sB + C * 4;             // [2 tiles][4 row chunks][H + 4]
  float *sU = sHsum + 2 * 4 * (H + 4);   // [8] upstream u per 32-sample chunk of the group
  float *sP = sU + 64;                   // [8 chunks][2 column halves] partial sums of w_o . h_L
  float *sMisc = sP + 64;                // [16] loss partials per warp
  float *sWq = sMisc + 16;               // [<= 8] quadrature weights of the group's rays (N_s >= 32)
  float *sY = sMisc + 24;                // [<= 8] measured data of the group's pixels
  uint64_t *bars = reinterpret_cast<uint64_t *>(sMisc + 64);
  uint64_t *a_full = bars, *acc_full = bars + 2, *sa_free = bars + 4;  // [2] each
  uint64_t *w_bar = bars + 6, *xb_bar = bars + 7, *xb_free = bars + 8;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 9);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  if (tid == EPI) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&a_full[s], kF2TileArrivals);
      mbar_init(&acc_full[s], 1);
      mbar_init(&sa_free[s], 2);  // MMA retired (tcgen05.commit) + bulk store done reading (copy warp)
    }
    mbar_init(w_bar, 1);
    mbar_init(xb_bar, 1);
    mbar_init(xb_free, 1);
    fence_mbar_init();
  }
  const int64_t per = (int64_t)H * H + H;
  for (int i = tid; i < (int)(LY::ONES + L * LY::BIAS_B) / 4; i += LY::NT) reinterpret_cast<uint32_t *>(sOnes)[i] = 0u;
  __syncthreads();
  for (int i = tid; i < 128; i += LY::NT) {
    *reinterpret_cast<__nv_bfloat16 *>(sOnes + nosw16_offset(i, 0)) = __float2bfloat16_rn(1.f);
    *reinterpret_cast<__nv_bfloat16 *>(sOnes + nosw16_offset(i, 1)) = __float2bfloat16_rn(1.f);
  }
  for (int i = tid; i < L * H; i += LY::NT) {
    const float hb = 0.5f * p.params[(i / H) * per + (int64_t)H * H + (i % H)];
    const __nv_bfloat16 hi = __float2bfloat16_rn(hb);
    const __nv_bfloat16 lo = __float2bfloat16_rn(hb - __bfloat162float(hi));
    uint8_t *bb = sBiasB + (size_t)(i / H) * LY::BIAS_B;
    *reinterpret_cast<__nv_bfloat16 *>(bb + nosw16_offset(i % H, 0)) = hi;
    *reinterpret_cast<__nv_bfloat16 *>(bb + nosw16_offset(i % H, 1)) = lo;
  }
  for (int i = tid; i <= H; i += LY::NT) sWo[i] = p.params[(int64_t)L * per + i];
  for (int i = tid; i < C * 4; i += LY::NT) sB[i] = p.B[i];
  if (H == 64)  // zero pad blocks after each A tile (rows 64..127 of the M = 128 dW operand)
    for (int i = tid; i < (int)(2 * TILE / 16); i += LY::NT) {
      const int s = i / (TILE / 16), k = i % (TILE / 16);
      reinterpret_cast<uint4 *>(sA0 + s * LY::A_BYTES + TILE)[k] = make_uint4(0, 0, 0, 0);
    }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t a0_base = smem_u32(sA0), xb_base = smem_u32(sXB), w_base = smem_u32(sW);
  const uint32_t ones_base = smem_u32(sOnes), biasb_base = smem_u32(sBiasB);
  const int64_t n_groups = (p.nsamp + 255) / 256;
  uint8_t *ring = p.ring + (size_t)blockIdx.x * 2 * (L + nf) * TILE;
  auto ring_s2 = [&](int slot, int l) { return ring + ((size_t)slot * (L + nf) + l) * TILE; };
  auto ring_h = [&](int slot, int j) { return ring + ((size_t)slot * (L + nf) + L + j) * TILE; };
  const uint64_t pol_keep = policy_evict_last(), pol_stream = policy_evict_first();

  if (tid >= EPI) {
    const uint8_t *wsrc = reinterpret_cast<const uint8_t *>(p.wpack_half);
    if (warp == EPI / 32 && lane == 0) {
      // ===================================================== MMA issuer (never blocks on copies)
      const uint32_t idf = idesc_bf16(128, H, 0, 0), idb = idesc_bf16(128, H, 0, 1), idw = idesc_bf16(128, H, 1, 1);
      if (L > 1) f2_ctl_wait(w_bar, 0);
      uint32_t aph[2] = {0, 0}, xph = 0, dw_init = 0;
      auto xb_wait = [&]() {
        f2_ctl_wait(xb_bar, xph);
        xph ^= 1;
        tc_fence_after();
      };
      for (int64_t gi = blockIdx.x; gi < n_groups; gi += gridDim.x) {
        for (int l = 0; l < L; ++l)
          for (int s = 0; s < 2; ++s) {
            const uint32_t a_base = a0_base + s * LY::A_BYTES;
            f2_ctl_wait(&a_full[s], aph[s]);
            aph[s] ^= 1;
            tc_fence_after();
            if (l == 0 && s == 0) xb_wait();  // W_0 of this group
            const uint32_t wl = l == 0 ? xb_base : w_base + (uint32_t)(l - 1) * LY::W_LAYER;
            umma_bf16(tmem + s * H, sdesc_none(ones_base, 128, 256), sdesc_none(biasb_base + l * LY::BIAS_B, 128, 256),
                      idf, 0u);
#pragma unroll
            for (int kk = 0; kk < H / 16; ++kk)
              umma_bf16(tmem + s * H, sdesc_sw128(a_base + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                        sdesc_sw128(wl + (kk >> 2) * (H * 128) + (kk & 3) * 32, 16, 1024), idf, 1u);
            umma_commit(&acc_full[s]);
            umma_commit(&sa_free[s]);
            if (l == 0 && s == 1) umma_commit(xb_free);  // W_0 retired for this group
          }
        for (int l = L - 1; l >= lmin; --l)
          for (int s = 0; s < 2; ++s) {
            const uint32_t a_base = a0_base + s * LY::A_BYTES;
            const bool fused = l >= nu;
            f2_ctl_wait(&a_full[s], aph[s]);
            aph[s] ^= 1;
            tc_fence_after();
            if (fused) {
              xb_wait();  // XB = h_{l-1} of this tile
              const uint32_t dwt = tmem + (uint32_t)(2 * H + (l - nu) * H);
              const uint32_t seen = (dw_init >> (l - nu)) & 1u;  // TMEM is not zeroed: first MMA overwrites
              dw_init |= 1u << (l - nu);
#pragma unroll
              for (int kk = 0; kk < 8; ++kk)
                umma_bf16(dwt, sdesc_sw128(a_base + kk * 2048, 16384, 1024), sdesc_sw128(xb_base + kk * 2048, 16384, 1024),
                          idw, (seen || kk > 0) ? 1u : 0u);
            }
            if (l > lmin) {
              const uint32_t wl = w_base + (uint32_t)(l - 1) * LY::W_LAYER;
#pragma unroll
              for (int kk = 0; kk < H / 16; ++kk)
                umma_bf16(tmem + s * H, sdesc_sw128(a_base + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                          sdesc_sw128(wl + kk * 2048, H * 128, 1024), idb, kk > 0);
            }
            umma_commit(&acc_full[s]);
            umma_commit(&sa_free[s]);
            if (fused) umma_commit(xb_free);
          }
      }
    } else if (warp == EPI / 32 + 1 && lane == 0) {
      // ===================================================== copy engine: weights, XB, ring / stash stores
      if (L > 1) {
        const uint32_t rb = (uint32_t)(L - 1) * LY::W_LAYER;
        mbar_arrive_expect_tx(w_bar, rb);
        for (uint32_t off = 0; off < rb; off += 32768u)
          bulk_g2s(sW + off, wsrc + LY::W_LAYER + off, min(32768u, rb - off), w_bar);
      }
      auto xb_load = [&](const void *src, uint32_t bytes, uint64_t pol) {
        mbar_arrive_expect_tx(xb_bar, bytes);
        for (uint32_t off = 0; off < bytes; off += 32768u)
          bulk_g2s_hint(sXB + off, reinterpret_cast<const uint8_t *>(src) + off, min(32768u, bytes - off), xb_bar, pol);
      };
      xb_load(wsrc, LY::W_LAYER, pol_keep);  // W_0 for the first group's forward
      uint32_t aph[2] = {0, 0}, fph = 0;
      auto free_wait = [&]() {
        f2_ctl_wait(xb_free, fph);
        fph ^= 1;
      };
      for (int64_t gi = blockIdx.x; gi < n_groups; gi += gridDim.x) {
        const bool more = gi + (int64_t)gridDim.x < n_groups;
        // ---------------------------------------------------------------- forward
        for (int l = 0; l < L; ++l)
          for (int s = 0; s < 2; ++s) {
            const int64_t tile = 2 * gi + s;
            uint8_t *sA = sA0 + s * LY::A_BYTES;
            f2_ctl_wait(&a_full[s], aph[s]);
            aph[s] ^= 1;
            if (l == L - 1 && s == 0 && l >= nu) {
              // the top layer's input of stream 0 is the first dW operand of the backward: into
              // XB as soon as W_0 has retired
              free_wait();
              bulk_s2g_hint(ring_h(0, l - nu), sA, TILE, pol_keep);
              bulk_commit();
              bulk_wait_all();
              xb_load(ring_h(0, l - nu), TILE, pol_stream);
            } else if (l >= nu) {
              bulk_s2g_hint(ring_h(s, l - nu), sA, TILE, pol_keep);
              bulk_commit();
              bulk_wait_read_all();
            } else if (l > 0 && !p.dw01) {
              // input of an unfused layer for K5 (which recomputes layer 0's features; k_dw01
              // recomputes both of its inputs)
              bulk_s2g_hint(p.hstash + ((size_t)l * p.n_tiles + tile) * TILE, sA, TILE, pol_stream);
              bulk_commit();
              bulk_wait_read_all();
            }
            mbar_arrive(&sa_free[s]);
          }
        // ---------------------------------------------------------------- backward
        for (int l = L - 1; l >= lmin; --l)
          for (int s = 0; s < 2; ++s) {
            const int64_t tile = 2 * gi + s;
            uint8_t *sA = sA0 + s * LY::A_BYTES;
            const bool fused = l >= nu;
            f2_ctl_wait(&a_full[s], aph[s]);
            aph[s] ^= 1;
            if (!fused) {
              bulk_s2g_hint(p.dstash + ((size_t)l * p.n_tiles + tile) * TILE, sA, TILE, pol_stream);
              bulk_commit();
              bulk_wait_read_all();
            }
            mbar_arrive(&sa_free[s]);
            if (fused) {  // next XB content, once this dW has retired
              const int ns = s == 0 ? 1 : 0, nl = s == 0 ? l : l - 1;
              free_wait();
              if (nl >= nu) {
                bulk_wait_all();  // the ring image was written by this thread's bulk store
                xb_load(ring_h(ns, nl - nu), TILE, pol_stream);
              } else if (more) {
                xb_load(wsrc, LY::W_LAYER, pol_keep);  // W_0 for the next group's forward
              }
            }
          }
      }
      bulk_wait_all();
    }
    __syncwarp();
  } else {
    // ===================================================== epilogue warpgroups
    const int s = tid >> 8;                  // stream / tile slot of the group
    const int wt = tid & 255;
    const int row = wt & 127, ch = wt >> 7;  // sample row, column half
    const uint32_t a_base = a0_base + s * LY::A_BYTES;
    uint32_t aoff[NCH][4];
#pragma unroll
    for (int c = 0; c < NCH; ++c)
#pragma unroll
      for (int q = 0; q < 4; ++q) aoff[c][q] = sw128_offset(row, ch * (H / 2) + c * 32 + 8 * q, 128);
    const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(s * H + ch * (H / 2));
    uint32_t accph = 0, sfph = 0;
    bool acc_pending = false;  // the previous group's last-step commit, consumed lazily
    bool sf_first = true;
#ifdef DINR_PHASES
    unsigned long long ph_acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, ph_t = clock64();
#define PH2(k)                                 \
  do {                                         \
    const unsigned long long _n = clock64();   \
    ph_acc[k] += _n - ph_t;                    \
    ph_t = _n;                                 \
  } while (0)
#else
#define PH2(k) \
  do {         \
  } while (0)
#endif
    auto wait_sa = [&]() {
      if (!sf_first) {
#ifdef DINR_PHASES
        const unsigned long long _w = clock64();
#endif
        f2_wait(&sa_free[s], sfph);
        sfph ^= 1;
#ifdef DINR_PHASES
        ph_acc[8] += clock64() - _w;
#endif
      }
      sf_first = false;
    };
    float dbacc[4][NCH];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int c = 0; c < NCH; ++c) dbacc[j][c] = 0.f;
    float wo_acc[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) wo_acc[c] = 0.f;
    float bo_acc = 0.f, loss_acc = 0.f;
    const int rays_per_group = 256 / p.n_s;
    const int pix_per_group = rays_per_group / p.S;
    // every tile holds whole pixels (S N_s <= 128): each stream combines its own pixels, no join.
    // Compiled in for H = 64 only (parallel64: -2.7 %); at H = 128 the extra code cost fan512 +1.9 %
    const bool sl = H == 64 && (128 % (p.S * p.n_s)) == 0;
    // loss operands: with sl each stream loads and stores its own tile's rays and pixels, so the
    // per-stream barrier orders them (stream 0 may start group gi+1 while stream 1 still forms the
    // loss of group gi when nothing else holds it back, e.g. L = 1); otherwise threads of stream 0
    // cover the group and the join barrier orders them
    const int pre_r = sl ? rays_per_group >> 1 : rays_per_group, pre_p = sl ? pix_per_group >> 1 : pix_per_group;
    const int pre_t = sl ? wt : tid, pre_ro = sl ? s * pre_r : 0, pre_po = sl ? s * pre_p : 0;

    for (int64_t gi = blockIdx.x; gi < n_groups; gi += gridDim.x) {
      const int64_t tile = 2 * gi + s;
      const int64_t g = tile * 128 + row;
      const bool valid = g < p.nsamp;
      // loss operands of the group's pixels (quadrature weights, measured data), fetched now so
      // that the loss phase -- where both streams wait -- has no global-memory latency
      float wq_pre = 0.f, y_pre = 0.f;  // loads in flight during the feature computation
      if (pre_t < pre_r) {
        const int64_t ray = gi * rays_per_group + pre_ro + pre_t;
        if (ray < p.n_pix * p.S) wq_pre = p.rec32[2 * ray + 1].w;
      }
      if (pre_t < pre_p) {
        const int64_t pix = gi * pix_per_group + pre_po + pre_t;
        if (pix < p.n_pix) y_pre = p.y[pix];
      }
      // ------------------------------------------------------------ a5/a6 features
      {
        const float4 rb = grff_coords(p.rec32, g, p.lg_ns, p.n_s, valid, p.jit);
        constexpr int NFC = (C / 2) / 8;  // 8-frequency chunks of this thread's half of the frequencies
        uint32_t pc[NFC][4], ps[NFC][4];
#pragma unroll
        for (int fc = 0; fc < NFC; ++fc) grff8(reinterpret_cast<const float4 *>(sB), ch * (C / 2) + 8 * fc, rb, pc[fc], ps[fc]);
        if (acc_pending) {  // the features above overlapped the previous group's last MMA
          f2_wait(&acc_full[s], accph);
          accph ^= 1;
          tc_fence_after();
          acc_pending = false;
        }
        wait_sa();
#pragma unroll
        for (int fc = 0; fc < NFC; ++fc) {
          const int c0 = ch * (C / 2) + 8 * fc;
          st_shared_v4(a_base + sw128_offset(row, c0, 128), pc[fc][0], pc[fc][1], pc[fc][2], pc[fc][3]);
          st_shared_v4(a_base + sw128_offset(row, C + c0, 128), ps[fc][0], ps[fc][1], ps[fc][2], ps[fc][3]);
        }
      }
      fence_proxy_async_smem();
      if (pre_t < pre_r) sWq[pre_ro + pre_t] = wq_pre;
      if (pre_t < pre_p) sY[pre_po + pre_t] = y_pre;
      PH2(0);
      f2_arrive_tile(&a_full[s], s);
      // ------------------------------------------------------------ a7/a8 forward layers
      float mu_part = 0.f;
      for (int l = 0; l < L; ++l) {
        const bool last = (l == L - 1);
        f2_wait(&acc_full[s], accph);
        accph ^= 1;
        tc_fence_after();
        PH2(1);
        // 16-column steps; the TMEM load of step k+1 is in flight while step k is computed
        constexpr int NHC = H / 32;  // 16-column steps in this thread's column half
        uint32_t va[16], vb[16];
        tmem_ld16(trow, va);
        tmem_wait_ld();
        reg_fence(va);
#pragma unroll
        for (int hc = 0; hc < NHC; ++hc) {
          uint32_t(&cur)[16] = (hc & 1) ? vb : va;
          uint32_t(&nxt)[16] = (hc & 1) ? va : vb;
#ifndef DINR_F2_NO_PREFETCH
          if (hc + 1 < NHC) tmem_ld16(trow + (hc + 1) * 16, nxt);
#else
          if (hc > 0) {
            tmem_ld16(trow + hc * 16, cur);
            tmem_wait_ld();
            reg_fence(cur);
          }
#endif
          const int col0 = ch * (H / 2) + hc * 16;
          uint32_t hpk[8], s2k[8];
#pragma unroll
          for (int i = 0; i < 16; i += 4) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const uint32_t yb = pack_bf16x2(__uint_as_float(cur[i + 2 * e]), __uint_as_float(cur[i + 2 * e + 1]));
              const uint32_t t = bf2_tanh(yb);
              hpk[i / 2 + e] = bf2_fma(yb, t, yb);
              const uint32_t w = bf2_fma(t, t ^ kBf2Sign, kBf2One);
              s2k[i / 2 + e] = bf2_fma(yb, w, bf2_add(t, kBf2One));
            }
          }
          if (last) {
            // top layer: s2 stays on chip, packed into this thread's already-consumed accumulator
            // columns (acc[s] is idle until the first backward dX MMA)
            tmem_st8(trow + hc * 8, s2k);
          } else if (l >= lmin) {
            // ring layout [16-column chunk][row][32 B]: one 256-bit store per thread, a warp covers
            // 1 KB contiguous
            st_global_v8_hint(ring_s2(s, l) + ((size_t)(col0 >> 4) * 128 + row) * 32, s2k, pol_keep);
          }
          if (!last) {
            if (hc == 0) wait_sa();
#pragma unroll
            for (int q = 0; q < 2; ++q)
              st_shared_v4(a_base + aoff[hc >> 1][(hc & 1) * 2 + q], hpk[4 * q], hpk[4 * q + 1], hpk[4 * q + 2],
                           hpk[4 * q + 3]);
          } else {
            float hv[16];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              hv[2 * i] = bf16lo(hpk[i]);
              hv[2 * i + 1] = bf16hi(hpk[i]);
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) mu_part = fmaf(sWo[col0 + i], hv[i], mu_part);
#ifndef DINR_F2_FP32_SUMS
            // column sums over the warp's 32 rows (lanes l and l^16 end with column l & 15): two
            // butterfly levels on packed bf16 pairs, then fp32
            uint32_t hw[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) hw[i] = hpk[i];
#pragma unroll
            for (int o = 4; o >= 2; o >>= 1) {  // lane bits 8, 4 <-> packed words 4, 2 apart
              const bool up = (lane & (2 * o)) != 0;
#pragma unroll
              for (int i = 0; i < o; ++i) {
                const uint32_t send = up ? hw[i] : hw[i + o];
                const uint32_t keep = up ? hw[i + o] : hw[i];
                hw[i] = bf2_add(keep, (uint32_t)__shfl_xor_sync(0xffffffffu, (int)send, 2 * o));
              }
            }
            hv[0] = bf16lo(hw[0]);
            hv[1] = bf16hi(hw[0]);
            hv[2] = bf16lo(hw[1]);
            hv[3] = bf16hi(hw[1]);
#pragma unroll
            for (int o = 2; o >= 1; o >>= 1) {
              const bool up = (lane & o) != 0;
#pragma unroll
              for (int i = 0; i < o; ++i) {
                float send = up ? hv[i] : hv[i + o];
                float keep = up ? hv[i + o] : hv[i];
                hv[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
              }
            }
#else
            // column sums over the warp's 32 rows in fp32 (lanes l and l^16 end with column l & 15):
            // four butterfly levels (lane bits 8 .. 1 <-> entries 8 .. 1 apart), then lane bit 16
#pragma unroll
            for (int o = 8; o >= 1; o >>= 1) {
              const bool up = (lane & o) != 0;
#pragma unroll
              for (int i = 0; i < o; ++i) {
                float send = up ? hv[i] : hv[i + o];
                float keep = up ? hv[i + o] : hv[i];
                hv[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
              }
            }
#endif
            hv[0] += __shfl_xor_sync(0xffffffffu, hv[0], 16);
            if (lane < 16) sHsum[(s * 4 + (warp & 3)) * (H + 4) + col0 + lane] = hv[0];
          }
#ifndef DINR_F2_NO_PREFETCH
          if (hc + 1 < NHC) {
            tmem_wait_ld();
            reg_fence(nxt);
          }
#endif
        }
        if (last) tmem_wait_st();
        tc_fence_before();
        if (!last) {
          fence_proxy_async_smem();
          f2_arrive_tile(&a_full[s], s);
        }
        PH2(2);
      }
      // ------------------------------------------------------------ a9-a11: combine + loss
      {  // 32-row partial sums of w_o . h_L per (chunk = tile s, lane quadrant; column half)
        float a = valid ? mu_part : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) sP[(s * 4 + (warp & 3)) * 2 + ch] = a;
      }
      if (sl)
        asm volatile("bar.sync %0, 256;" ::"r"(2 + s) : "memory");
      else
        named_sync(1, EPI);
      // a9-a11 on warp 0: lane q < 8 = ray chunk q of the group (32 samples).  S * N_s divides 256
      // and both are powers of two, so a ray is an aligned group of cpr = N_s / 32 lanes and a pixel
      // an aligned group of S * cpr lanes: ray sums, the Beer's-law min / sum and the pixel's
      // upstream factors are xor-butterflies inside those groups.
      // (sl: the first warp of each stream does its own tile's chunks 4s..4s+3 on lanes 0-3; pixels
      // then span <= 4 chunks, so only the butterfly levels 1, 2 act)
      if (sl ? (warp & 7) == 0 : warp == 0) {
        // powers of two throughout: shifts and masks, no integer or fp32 divisions on the join
        const int lg_cpr = p.lg_ns - 5, lg_s = __ffs(p.S) - 1;
        const int nq = sl ? 4 : 8;
        const int q = sl ? 4 * s + (lane & 3) : (lane & 7), cpr = 1 << lg_cpr, gl = cpr << lg_s;
        const int ray_l = q >> lg_cpr, pix_l = ray_l >> lg_s;
        const int64_t pix = gi * pix_per_group + pix_l;
        const bool live = lane < nq && pix < p.n_pix;
        const float inv_s = __int_as_float((127 - lg_s) << 23);  // 1 / S exactly
        float a = sP[2 * q] + sP[2 * q + 1] + 32.f * sWo[H];  // chunk sum of w_o . h_L + b_o
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {  // the three butterfly levels, each used inside its group only
          const float t = __shfl_xor_sync(0xffffffffu, a, o);
          if (o < cpr) a += t;
        }
        const float wq = sWq[ray_l];  // prefetched at the start of the group
        const float pv = wq > 0.f ? wq * (p.mu0 * a) : 0.f;
        const bool beer = p.combine != DINR_LINEAR;
        float m = pv;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
          const float t = __shfl_xor_sync(0xffffffffu, m, o);
          if (o >= cpr && o < gl) m = fminf(m, t);
        }
        const float e = beer ? __expf(m - pv) : pv;
        float sum = (q & (cpr - 1)) == 0 ? e : 0.f;  // one term per ray
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
          const float t = __shfl_xor_sync(0xffffffffu, sum, o);
          if (o < gl) sum += t;
        }
        const float T = sum * inv_s;
        const float fh = beer ? m - __logf(T) : T;
        const bool leader = live && (q & (gl - 1)) == 0;
        if (leader && p.fhat) p.fhat[pix] = fh;
        const float res = sY[pix_l] - fh;
        if (leader) loss_acc += res * res;
        const float gg = -2.f * res * p.inv_n;
        const float pi = beer ? __fdividef(e, sum) : inv_s;  // e^{-(p - m)} / (S T)
        if (lane < nq) sU[q] = live ? gg * pi * wq * p.mu0 : 0.f;
      }
      if (sl)
        asm volatile("bar.sync %0, 256;" ::"r"(2 + s) : "memory");
      else
        named_sync(1, EPI);
      // head gradients (warps 0 and 4 of warpgroup 0 own all H columns; with sl each stream's warps
      // 0 and 4 accumulate its own chunks, combined at the flush)
      if ((sl || s == 0) && (warp & 3) == 0) {
        const int q0 = sl ? 4 * s : 0, q1 = sl ? 4 * s + 4 : 8;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          const int col = ch * (H / 2) + c * 32 + lane;
          float a = 0.f;
          for (int q = q0; q < q1; ++q) a += sU[q] * sHsum[q * (H + 4) + col];
          wo_acc[c] += a;
        }
      }
      if (wt == 0 && (sl || s == 0)) {
        const int q0 = sl ? 4 * s : 0, q1 = sl ? 4 * s + 4 : 8;
        float a = 0.f;
        for (int q = q0; q < q1; ++q)
          if (gi * 256 + q * 32 < p.nsamp) a += 32.f * sU[q];
        bo_acc += a;
      }
      // ------------------------------------------------------------ a12 backward
      const float u_row = sU[s * 4 + (row >> 5)];
      PH2(3);
      uint4 sq[NCH][4];
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < NCH; ++c) {  // top-layer s2 from TMEM (stored by the last forward epilogue)
        uint32_t w[16];
        tmem_ld16(trow + c * 16, w);
        tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 4; ++q) sq[c][q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
      }
      for (int l = L - 1; l >= lmin; --l) {
        const bool top = (l == L - 1);
        if (!top) {
          f2_wait(&acc_full[s], accph);
          accph ^= 1;
          tc_fence_after();
          PH2(4);
        }
        uint32_t dp[NCH][16];
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          const int col0 = ch * (H / 2) + c * 32;
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            uint32_t v[16];
            if (!top) {
              tmem_ld16(trow + c * 32 + hf * 16, v);
              tmem_wait_ld();
            }
#pragma unroll
            for (int q2 = 0; q2 < 2; ++q2) {
              const uint4 w = sq[c][hf * 2 + q2];
              const uint32_t w4[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int i = q2 * 8 + 2 * e;
                const int cc = hf * 16 + i;
                const float e0 = top ? 0.5f * u_row * sWo[col0 + cc] : __uint_as_float(v[i]);
                const float e1 = top ? 0.5f * u_row * sWo[col0 + cc + 1] : __uint_as_float(v[i + 1]);
#ifdef DINR_F2_PACKED_DELTA
                dp[c][cc / 2] = bf2_mul(pack_bf16x2(e0, e1), w4[e]);
#else  // delta = e * swish'(z) in fp32, one bf16 rounding (the MMA operand)
                dp[c][cc / 2] = pack_bf16x2(e0 * bf16lo(w4[e]), e1 * bf16hi(w4[e]));
#endif
              }
            }
          }
        }
        tc_fence_before();
        wait_sa();
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            st_shared_v4(a_base + aoff[c][q], dp[c][4 * q], dp[c][4 * q + 1], dp[c][4 * q + 2], dp[c][4 * q + 3]);
        fence_proxy_async_smem();
        PH2(5);
        f2_arrive_tile(&a_full[s], s);
        if (l > lmin) {  // prefetch s2 of the next backward step
#pragma unroll
          for (int c = 0; c < NCH; ++c)
#pragma unroll
            for (int hf = 0; hf < 2; ++hf)
              ld_global_v8_hint(ring_s2(s, l - 1) + ((size_t)((ch * (H / 2) + c * 32 + hf * 16) >> 4) * 128 + row) * 32,
                                sq[c][2 * hf], sq[c][2 * hf + 1], pol_stream);
        }
        if (l >= nu) {  // db of a fused layer: column sums of delta over the warp's 32 rows
#pragma unroll
          for (int c = 0; c < NCH; ++c) {
#ifndef DINR_F2_FP32_SUMS
            // transpose-reduce: the first two butterfly levels on packed bf16 pairs (sums of 2
            // and 4 rows), the last three in fp32; lane l ends with column l's 32-row sum
            uint32_t w[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) w[i] = dp[c][i];
#pragma unroll
            for (int o = 8; o >= 4; o >>= 1) {  // lane bits 16, 8 <-> packed words 8, 4 apart
              const bool up = (lane & (2 * o)) != 0;
#pragma unroll
              for (int i = 0; i < o; ++i) {
                const uint32_t send = up ? w[i] : w[i + o];
                const uint32_t keep = up ? w[i + o] : w[i];
                w[i] = bf2_add(keep, (uint32_t)__shfl_xor_sync(0xffffffffu, (int)send, 2 * o));
              }
            }
            float d[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              d[2 * i] = bf16lo(w[i]);
              d[2 * i + 1] = bf16hi(w[i]);
            }
#pragma unroll
            for (int o = 4; o >= 1; o >>= 1) {
              const bool up = (lane & o) != 0;
#pragma unroll
              for (int i = 0; i < o; ++i) {
                float send = up ? d[i] : d[i + o];
                float keep = up ? d[i + o] : d[i];
                d[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
              }
            }
#else
            // transpose-reduce in fp32 (five butterfly levels, lane bits 16 .. 1 <-> entries 16 .. 1
            // apart); lane l ends with column l's 32-row sum
            float d[32];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              d[2 * i] = bf16lo(dp[c][i]);
              d[2 * i + 1] = bf16hi(dp[c][i]);
            }
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) {
              const bool up = (lane & o) != 0;
#pragma unroll
              for (int i = 0; i < o; ++i) {
                float send = up ? d[i] : d[i + o];
                float keep = up ? d[i + o] : d[i];
                d[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
              }
            }
#endif
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (j == l - nu) dbacc[j][c] += d[0];
          }
        }
        PH2(6);
      }
      // the last step (dW MMA or delta stash store) must retire before A_s is rewritten: its commit
      // is consumed after the next group's features are computed (wait_sa there covers A_s)
      acc_pending = true;
      PH2(7);
    }
    if (acc_pending) {  // every MMA retired before the TMEM dW accumulators are read out
      f2_wait(&acc_full[s], accph);
      accph ^= 1;
      tc_fence_after();
    }
    // ------------------------------------------------------------ flush per-CTA partials
#ifdef DINR_PHASES
    if (wt == 0 && p.dbg)
      for (int k = 0; k < 9; ++k) p.dbg[(size_t)blockIdx.x * 32 + s * 16 + k] = ph_acc[k];
#endif
#undef PH2
    named_sync(1, EPI);
    for (int j = 0; j < nf; ++j) {
      if (s != (j & 1)) continue;  // warpgroup j%2 flushes fused layer j
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const int col0 = ch * (H / 2) + c * 32;
        uint32_t v[32];
        tmem_ld32(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(2 * H + j * H + col0), v);
        tmem_wait_ld();
        if (H >= 128 || row < 64) {
          float *dst = p.dw_part + (((size_t)j * gridDim.x + blockIdx.x) * 128 + row) * H + col0;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            reinterpret_cast<float4 *>(dst)[q] = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                                             __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]));
        }
      }
    }
    float *red = sHsum;  // reuse: [2 streams][4 row chunks][H + 4]
#pragma unroll
    for (int j = 0; j < 4; ++j) {  // static j: dbacc stays in registers
      if (j >= nf) break;
      named_sync(1, EPI);
#pragma unroll
      for (int c = 0; c < NCH; ++c) red[(s * 4 + (warp & 3)) * (H + 4) + ch * (H / 2) + c * 32 + lane] = dbacc[j][c];
      named_sync(1, EPI);
      if (tid < H) {
        float a = 0.f;
        for (int w = 0; w < 8; ++w) a += red[w * (H + 4) + tid];
        p.db_part[((size_t)j * gridDim.x + blockIdx.x) * 128 + tid] = a;
      }
    }
    named_sync(1, EPI);
    if (sl) {  // stream 1's head partials (its own chunks) onto stream 0's
      if (s == 1 && (warp & 3) == 0)
#pragma unroll
        for (int c = 0; c < NCH; ++c) red[ch * (H / 2) + c * 32 + lane] = wo_acc[c];
      if (s == 1 && wt == 0) red[H] = bo_acc;
      named_sync(1, EPI);
      if (s == 0 && (warp & 3) == 0)
#pragma unroll
        for (int c = 0; c < NCH; ++c) wo_acc[c] += red[ch * (H / 2) + c * 32 + lane];
      if (tid == 0) bo_acc += red[H];
    }
    if (s == 0 && (warp & 3) == 0) {
#pragma unroll
      for (int c = 0; c < NCH; ++c) p.head_part[(size_t)blockIdx.x * (H + 1) + ch * (H / 2) + c * 32 + lane] = wo_acc[c];
    }
    if (tid == 0) p.head_part[(size_t)blockIdx.x * (H + 1) + H] = bo_acc;
    for (int o = 16; o > 0; o >>= 1) loss_acc += __shfl_xor_sync(0xffffffffu, loss_acc, o);
    if (lane == 0) sMisc[warp] = loss_acc;
    named_sync(1, EPI);
    if (tid == 0) {
      float a = 0.f;
      for (int w = 0; w < EPI / 32; ++w) a += sMisc[w];
      p.loss_part[blockIdx.x] = a;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace dinr
