// k_fused.cuh -- fused training step for pixel groups that fit two 128-sample tiles
// (256 % (S*N_s) == 0, H <= 128): forward of both tiles -> in-CTA combine + loss (the K4
// math) -> backward of both tiles, with the weight gradients of the top `nf` layers
// accumulated in TMEM for the CTA's whole lifetime.  Replaces K2 + K4 + K3 (and most of K5)
// for these workloads (north_star subsystems (2)-(4)).
//
// Roles: CG = H/32 column groups; 128*CG epilogue threads (thread owns TMEM lane = sample row
// r = tid % 128 and the 32 columns of group tid / 128), then one control warp whose lane 0
// issues every tcgen05.mma and bulk copy.
// TMEM: [0, H) working accumulator; [H + j*H, H + (j+1)*H) dW of layer nu + j (fp32).
// Weights are the 0.5-prescaled bf16 images (exact): the forward MMA yields y = z/2 and
//   h = swish(z) = y (1 + tanh y),   s2 = 2 swish'(z) = 1 + t + y (1 - t^2),  t = tanh y;
// the backward dX MMA on the same image yields e/2, so delta = (e/2) * s2.
// Per-tile state between forward and backward (s2 of every layer, h of the fused layers) goes
// through a small per-CTA global ring kept in L2 with an evict_last policy.
#pragma once
#include "internal.cuh"
#include "ptx_sm100.cuh"
#include "k_features.cuh"

namespace dinr {

struct FusedParams {
  const float4 *rec32;
  int64_t n_pix, nsamp;
  int n_s, lg_ns, S, L, nf;  // nf = number of top layers whose dW is fused in TMEM
  int combine;
  float mu0, inv_n;
  const float *params;    // fp32 D5
  const float *B;         // C x 4
  const uint16_t *wpack_half;  // 0.5-scaled SW128 images
  const float *y;         // measured projections [n_pix]
  float *fhat;            // [n_pix] or null
  uint8_t *ring;          // per CTA: 2 slots x (L s2 tiles + nf h tiles) x H*256 bytes
  uint8_t *hstash, *dstash;  // unfused layers [L-nf][n_tiles] tile images (K5 operands)
  int64_t n_tiles;
  float *dw_part;         // [nf][grid][128][H]
  float *db_part;         // [nf][grid][128]
  float *head_part;       // [grid][H+1]
  float *loss_part;       // [grid]
  Jitter jit;                // N3 sample placement
  int dw01;                  // layer 1's input is recomputed after the kernel (k_dw01): no h stash
  unsigned long long *dbg;  // DINR_PHASES builds: [grid][8] cycle counters
};

template <int H>
struct FusedLayout {
  static constexpr int CG = H / 32;                // column groups = epilogue warpgroups
  static constexpr int EPI = 128 * CG;             // epilogue threads
  static constexpr int NT = EPI + 32;              // + control warp
  static constexpr uint32_t TILE = H * 256u;       // one 128-row bf16 tile image
  static constexpr uint32_t A_BYTES = H == 64 ? 2 * TILE : TILE;  // H = 64: zero pad block for M = 128 dW
  static constexpr uint32_t W_LAYER = H * H * 2u;
  static size_t smem_bytes(int L) {
    return 1024 + A_BYTES + TILE + (size_t)L * W_LAYER + (size_t)L * H * 4 + (H + 4) * 4 + (H / 2) * 16 +
           2 * 4 * (H + 4) * 4 + 2 * 128 * CG * 4 + 3 * 64 * 4 + 256;
  }
};

#ifdef DINR_PHASES
#define PH_MARK(k)                        \
  do {                                    \
    if (tid == 0) {                       \
      unsigned long long _t = clock64();  \
      ph[k] += _t - ph_last;              \
      ph_last = _t;                       \
    }                                     \
  } while (0)
#else
#define PH_MARK(k) \
  do {             \
  } while (0)
#endif

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int H>
__global__ void __launch_bounds__(FusedLayout<H>::NT, 1) k_fused(FusedParams p) {
  using LY = FusedLayout<H>;
  constexpr int C = H / 2;
  constexpr int CG = LY::CG;
  constexpr int EPI = LY::EPI;
  constexpr uint32_t TILE = LY::TILE;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared address space
  const int L = p.L, nf = p.nf, nu = L - nf;  // unfused layers: 0..nu-1
  uint8_t *sA = smem;
  uint8_t *sHB = sA + LY::A_BYTES;
  uint8_t *sW = sHB + TILE;
  float *sBias = reinterpret_cast<float *>(sW + (size_t)L * LY::W_LAYER);  // 0.5 * b_l
  float *sWo = sBias + L * H;                                              // w_o[H], b_o
  float *sB = sWo + H + 4;                                                 // C x 4
  float *sHsum = sB + C * 4;             // [2 tiles][4 row chunks][H + 4]: sum of h_L over 32 rows
  float *sMu = sHsum + 2 * 4 * (H + 4);  // [2 tiles][128 rows][CG]
  float *sU = sMu + 2 * 128 * CG;        // [8] upstream u per 32-sample chunk of the group
  float *sP = sU + 64;                   // [8] chunk sums of M
  float *sMisc = sP + 64;                // [warps] loss partials
  uint64_t *bars = reinterpret_cast<uint64_t *>(sMisc + 64);
  uint64_t *a_full = bars, *acc_full = bars + 1, *w_bar = bars + 2, *hb_bar = bars + 3, *sa_free = bars + 4;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 5);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool ctrl = (tid >= EPI);
  if (warp == 0) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  if (tid == EPI) {
    mbar_init(a_full, EPI);
    mbar_init(acc_full, 1);
    mbar_init(w_bar, 1);
    mbar_init(hb_bar, 1);
    mbar_init(sa_free, 1);
    fence_mbar_init();
  }
  const int64_t per = (int64_t)H * H + H;
  for (int i = tid; i < L * H; i += LY::NT) sBias[i] = 0.5f * p.params[(i / H) * per + (int64_t)H * H + (i % H)];
  for (int i = tid; i <= H; i += LY::NT) sWo[i] = p.params[(int64_t)L * per + i];
  for (int i = tid; i < C * 4; i += LY::NT) sB[i] = p.B[i];
  if (H == 64)  // zero pad block after the A tile (rows 64..127 of the M = 128 dW operand)
    for (int i = tid; i < (int)(TILE / 16); i += LY::NT) reinterpret_cast<uint4 *>(sA + TILE)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t a_base = smem_u32(sA), hb_base = smem_u32(sHB), w_base = smem_u32(sW);
  const int64_t n_groups = (p.nsamp + 255) / 256;
  uint8_t *ring = p.ring + (size_t)blockIdx.x * 2 * (L + nf) * TILE;
  auto ring_s2 = [&](int slot, int l) { return ring + ((size_t)slot * (L + nf) + l) * TILE; };
  auto ring_h = [&](int slot, int j) { return ring + ((size_t)slot * (L + nf) + L + j) * TILE; };
  const uint64_t pol_keep = policy_evict_last(), pol_stream = policy_evict_first();

  if (ctrl) {
    // ===================================================== MMA issuer / copy engine
    if (lane == 0) {
      const uint32_t idf = idesc_bf16(128, H, 0, 0), idb = idesc_bf16(128, H, 0, 1), idw = idesc_bf16(128, H, 1, 1);
      mbar_arrive_expect_tx(w_bar, (uint32_t)L * LY::W_LAYER);
      for (uint32_t off = 0; off < (uint32_t)L * LY::W_LAYER; off += 32768u)
        bulk_g2s(sW + off, reinterpret_cast<const uint8_t *>(p.wpack_half) + off,
                 min(32768u, (uint32_t)L * LY::W_LAYER - off), w_bar);
      mbar_wait(w_bar, 0);
      uint32_t aph = 0, hph = 0, ncommit = 0, dw_init = 0;
      for (int64_t gi = blockIdx.x; gi < n_groups; gi += gridDim.x) {
        for (int s = 0; s < 2; ++s) {
          const int64_t tile = 2 * gi + s;
          for (int l = 0; l < L; ++l) {
            mbar_wait(a_full, aph);
            aph ^= 1;
            tc_fence_after();
            // h_l (the A tile) is an operand of dW_l: fused -> L2 ring, unfused -> dW GEMM stash
            if (l >= nu)
              bulk_s2g_hint(ring_h(s, l - nu), sA, TILE, pol_keep);
            else if (l > 0)  // layer 0's input (the GRFF features) is recomputed by the dW GEMM
              bulk_s2g_hint(p.hstash + ((size_t)l * p.n_tiles + tile) * TILE, sA, TILE, pol_stream);
            bulk_commit();
            const uint32_t wl = w_base + (uint32_t)l * LY::W_LAYER;
#pragma unroll
            for (int kk = 0; kk < H / 16; ++kk)
              umma_bf16(tmem, sdesc_sw128(a_base + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                        sdesc_sw128(wl + (kk >> 2) * (H * 128) + (kk & 3) * 32, 16, 1024), idf, kk > 0);
            umma_commit(acc_full);
            ++ncommit;
            bulk_wait_read_all();  // the copy engine is done with sA
            mbar_arrive(sa_free);
          }
        }
        // backward (the loss runs on the epilogue warps in between)
        for (int s = 0; s < 2; ++s) {
          const int64_t tile = 2 * gi + s;
          for (int l = L - 1; l >= 0; --l) {
            const bool fused = l >= nu;
            if (fused) {  // prefetch h_l into HB (HB is free: the previous dW MMA retired)
              mbar_arrive_expect_tx(hb_bar, TILE);
              bulk_g2s_hint(sHB, ring_h(s, l - nu), TILE, hb_bar, pol_stream);
            }
            mbar_wait(a_full, aph);
            aph ^= 1;
            tc_fence_after();
            if (!fused) {  // delta_l image for the dW GEMM
              bulk_s2g_hint(p.dstash + ((size_t)l * p.n_tiles + tile) * TILE, sA, TILE, pol_stream);
              bulk_commit();
            }
            if (fused) {
              mbar_wait(hb_bar, hph);
              hph ^= 1;
              tc_fence_after();
              const uint32_t dwt = tmem + (uint32_t)(H + (l - nu) * H);
              const uint32_t seen = (dw_init >> (l - nu)) & 1u;  // TMEM is not zeroed: first MMA overwrites
              dw_init |= 1u << (l - nu);
#pragma unroll
              for (int kk = 0; kk < 8; ++kk)
                umma_bf16(dwt, sdesc_sw128(a_base + kk * 2048, 16384, 1024), sdesc_sw128(hb_base + kk * 2048, 16384, 1024),
                          idw, (seen || kk > 0) ? 1u : 0u);
            }
            if (l > 0) {
              const uint32_t wl = w_base + (uint32_t)l * LY::W_LAYER;
#pragma unroll
              for (int kk = 0; kk < H / 16; ++kk)
                umma_bf16(tmem, sdesc_sw128(a_base + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                          sdesc_sw128(wl + kk * 2048, H * 128, 1024), idb, kk > 0);
            }
            umma_commit(acc_full);
            ++ncommit;
            bulk_wait_read_all();
            mbar_arrive(sa_free);
            // HB is reused by the next fused layer: wait until this dW MMA has retired
            if (fused) mbar_wait(acc_full, (ncommit - 1) & 1);
          }
        }
      }
      bulk_wait_all();
    }
    __syncwarp();
  } else {
    // ===================================================== epilogue warps
    const int row = tid & 127, cg = tid >> 7;
    const int col0 = cg * 32;
    uint32_t aoff[4];  // SW128 byte offsets of this thread's four 16-B chunks in a tile image
#pragma unroll
    for (int q = 0; q < 4; ++q) aoff[q] = sw128_offset(row, col0 + 8 * q, 128);
    const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)col0;
    uint32_t accph = 0;
    uint32_t sfph = 0;
    bool sf_first = true;
    auto wait_sa = [&]() {  // the copy engine has finished reading sA for the previous step
      if (!sf_first) {
        mbar_wait_sleep(sa_free, sfph);
        sfph ^= 1;
      }
      sf_first = false;
    };
#ifdef DINR_PHASES
    unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0}, ph_last = clock64();
#endif
    float dbacc[4] = {0.f, 0.f, 0.f, 0.f};  // fused-layer bias gradients (lane = column)
    float wo_acc = 0.f;                      // dL/dw_o partial (warps with warp % 4 == 0)
    float bo_acc = 0.f, loss_acc = 0.f;
    const int rays_per_group = 256 / p.n_s;
    const int pix_per_group = rays_per_group / p.S;
    const int chunks_per_ray = p.n_s / 32;

    for (int64_t gi = blockIdx.x; gi < n_groups; gi += gridDim.x) {
      // ------------------------------------------------------------ forward, two tiles
      for (int s = 0; s < 2; ++s) {
        const int64_t tile = 2 * gi + s;
        const int64_t g = tile * 128 + row;
        const bool valid = g < p.nsamp;
        {  // a5/a6: sample point, normalization and GRFF features of this thread's 16 frequencies
          const float4 rb = grff_coords(p.rec32, g, p.lg_ns, p.n_s, valid, p.jit);  // N_s is a power of two here
          constexpr int NCH = (C / CG) / 8;  // 8-frequency chunks per thread
          uint32_t pc[NCH][4], ps[NCH][4];
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) grff8(reinterpret_cast<const float4 *>(sB), cg * (C / CG) + 8 * ch, rb, pc[ch], ps[ch]);
          wait_sa();
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) {
            const int c0 = cg * (C / CG) + 8 * ch;
            st_shared_v4(a_base + sw128_offset(row, c0, 128), pc[ch][0], pc[ch][1], pc[ch][2], pc[ch][3]);
            st_shared_v4(a_base + sw128_offset(row, C + c0, 128), ps[ch][0], ps[ch][1], ps[ch][2], ps[ch][3]);
          }
        }
        fence_proxy_async_smem();
        mbar_arrive(a_full);
        PH_MARK(0);
        float mu_part = 0.f;
        for (int l = 0; l < L; ++l) {
          const bool last = (l == L - 1);
          PH_MARK(2);
          mbar_wait_sleep(acc_full, accph);
          PH_MARK(1);
          accph ^= 1;
          tc_fence_after();
          uint32_t hpk[16], s2k[16];  // packed bf16x2 results for this thread's 32 columns
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            uint32_t v[16];
            tmem_ld16(trow + hf * 16, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; i += 4) {
              const float4 b4 = *reinterpret_cast<const float4 *>(sBias + l * H + col0 + hf * 16 + i);
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                // h = y (1 + tanh y), s2 = 1 + t + y (1 - t^2) in packed bf16x2
                const float bb0 = e ? b4.z : b4.x, bb1 = e ? b4.w : b4.y;
                const uint32_t yb = pack_bf16x2(__uint_as_float(v[i + 2 * e]) + bb0, __uint_as_float(v[i + 2 * e + 1]) + bb1);
                const uint32_t t = bf2_tanh(yb);
                hpk[(hf * 16 + i) / 2 + e] = bf2_fma(yb, t, yb);
                const uint32_t w = bf2_fma(t, t ^ kBf2Sign, kBf2One);
                s2k[(hf * 16 + i) / 2 + e] = bf2_fma(yb, w, bf2_add(t, kBf2One));
              }
            }
          }
          tc_fence_before();
          if (!last) {
            wait_sa();
#pragma unroll
            for (int q = 0; q < 4; ++q)
              st_shared_v4(a_base + aoff[q], hpk[4 * q], hpk[4 * q + 1], hpk[4 * q + 2], hpk[4 * q + 3]);
#ifndef DINR_EXP_NO_FENCE
            fence_proxy_async_smem();
#endif
            mbar_arrive(a_full);
          }
#ifndef DINR_EXP_NO_S2_STORE
          uint4 *s2dst = reinterpret_cast<uint4 *>(ring_s2(s, l));
#pragma unroll
          for (int q = 0; q < 4; ++q)
            st_global_v4_hint(s2dst + (size_t)((col0 >> 3) + q) * 128 + row,
                              make_uint4(s2k[4 * q], s2k[4 * q + 1], s2k[4 * q + 2], s2k[4 * q + 3]), pol_keep);
#endif
          if (last) {
            float hv[32];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              hv[2 * i] = bf16lo(hpk[i]);
              hv[2 * i + 1] = bf16hi(hpk[i]);
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) mu_part = fmaf(sWo[col0 + i], hv[i], mu_part);
            // sum of h_L over this warp's 32 rows (transpose-reduce: lane i gets column col0+i)
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) {
              const bool up = (lane & o) != 0;
#pragma unroll
              for (int i = 0; i < o; ++i) {
                float send = up ? hv[i] : hv[i + o];
                float keep = up ? hv[i + o] : hv[i];
                hv[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
              }
            }
            sHsum[(s * 4 + (warp & 3)) * (H + 4) + col0 + lane] = valid ? hv[0] : 0.f;
          }
        }
        sMu[(s * 128 + row) * CG + cg] = valid ? mu_part : 0.f;
      }
      // ------------------------------------------------------------ a9-a11: combine + loss
      fence_proxy_async_global();  // ring h images (generic stores) are read back by TMA below
      named_sync(1, EPI);
      if (warp < 8) {  // a9: chunk sums of M = mu0 (w_o . h_L + b_o), warp q <-> 32-sample chunk q
        const int ss = warp >> 2, rr = (warp & 3) * 32 + lane;
        float m = sWo[H];
#pragma unroll
        for (int c = 0; c < CG; ++c) m += sMu[(ss * 128 + rr) * CG + c];
        float a = ((2 * gi + ss) * 128 + rr < p.nsamp) ? p.mu0 * m : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) sP[warp] = a;
      }
      named_sync(1, EPI);
      if (tid < pix_per_group) {
        const int64_t pix = gi * pix_per_group + tid;
        if (pix < p.n_pix) {
          float pv[8], wqv[8];
          for (int s = 0; s < p.S; ++s) {
            const int ray_l = tid * p.S + s;
            const int64_t ray = pix * p.S + s;
            wqv[s] = p.rec32[2 * ray + 1].w;
            float acc = 0.f;
            for (int c = 0; c < chunks_per_ray; ++c) acc += sP[ray_l * chunks_per_ray + c];
            pv[s] = wqv[s] > 0.f ? wqv[s] * acc : 0.f;
          }
          float fh, T = 1.f, m = 0.f;
          if (p.combine == DINR_LINEAR) {
            float acc = 0.f;
            for (int s = 0; s < p.S; ++s) acc += pv[s];
            fh = acc / (float)p.S;
          } else {
            m = pv[0];
            for (int s = 1; s < p.S; ++s) m = fminf(m, pv[s]);
            float acc = 0.f;
            for (int s = 0; s < p.S; ++s) acc += expf(-(pv[s] - m));
            T = acc / (float)p.S;
            fh = m - logf(T);
          }
          if (p.fhat) p.fhat[pix] = fh;
          const float res = p.y[pix] - fh;
          loss_acc += res * res;
          const float gg = -2.f * res * p.inv_n;
          for (int s = 0; s < p.S; ++s) {
            float pi = p.combine == DINR_LINEAR ? 1.f / (float)p.S : expf(-(pv[s] - m)) / ((float)p.S * T);
            const float us = gg * pi * wqv[s] * p.mu0;
            for (int c = 0; c < chunks_per_ray; ++c) sU[(tid * p.S + s) * chunks_per_ray + c] = us;
          }
        } else {
          for (int s = 0; s < p.S; ++s)
            for (int c = 0; c < chunks_per_ray; ++c) sU[(tid * p.S + s) * chunks_per_ray + c] = 0.f;
        }
      }
      named_sync(1, EPI);
      PH_MARK(3);
      // head gradients: dL/dw_o += sum_chunks u_chunk hsum_chunk, dL/db_o += sum u over samples
      if ((warp & 3) == 0) {
        float a = 0.f;
#pragma unroll
        for (int q = 0; q < 8; ++q) a += sU[q] * sHsum[q * (H + 4) + col0 + lane];
        wo_acc += a;
      }
      if (tid == 0) {
        float a = 0.f;
        for (int q = 0; q < 8; ++q)
          if (gi * 256 + q * 32 < p.nsamp) a += 32.f * sU[q];
        bo_acc += a;
      }
      // ------------------------------------------------------------ a12: backward, two tiles
      uint4 sq[4];  // s2 of the current backward step, prefetched one step ahead (L2 latency)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        sq[q] = ld_global_v4_hint(reinterpret_cast<const uint4 *>(ring_s2(0, L - 1)) + (size_t)((col0 >> 3) + q) * 128 + row,
                                  pol_stream);
      for (int s = 0; s < 2; ++s) {
        const float u_row = sU[s * 4 + (row >> 5)];
        for (int l = L - 1; l >= 0; --l) {
          const bool top = (l == L - 1);
          if (!top) {
            PH_MARK(6);
            mbar_wait_sleep(acc_full, accph);
            PH_MARK(5);
            accph ^= 1;
            tc_fence_after();
          }
          uint32_t dp[16];  // delta = (e/2) * s2 in packed bf16x2
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            uint32_t v[16];
            if (!top) {
              tmem_ld16(trow + hf * 16, v);
              tmem_wait_ld();
            }
#pragma unroll
            for (int q2 = 0; q2 < 2; ++q2) {
              const uint4 w = sq[hf * 2 + q2];
              const uint32_t w4[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int i = q2 * 8 + 2 * e;  // column within the 16-column half
                const int c = hf * 16 + i;
                float e0 = top ? 0.5f * u_row * sWo[col0 + c] : __uint_as_float(v[i]);
                float e1 = top ? 0.5f * u_row * sWo[col0 + c + 1] : __uint_as_float(v[i + 1]);
#ifdef DINR_F2_PACKED_DELTA
                dp[c / 2] = bf2_mul(pack_bf16x2(e0, e1), w4[e]);
#else  // delta in fp32, one bf16 rounding (as k_fused2)
                dp[c / 2] = pack_bf16x2(e0 * bf16lo(w4[e]), e1 * bf16hi(w4[e]));
#endif
              }
            }
          }
          tc_fence_before();
          wait_sa();
#pragma unroll
          for (int q = 0; q < 4; ++q)
            st_shared_v4(a_base + aoff[q], dp[4 * q], dp[4 * q + 1], dp[4 * q + 2], dp[4 * q + 3]);
          fence_proxy_async_smem();
          mbar_arrive(a_full);
          PH_MARK(4);
          {  // prefetch s2 of the next backward step
            const int ns = l > 0 ? s : s + 1, nl = l > 0 ? l - 1 : L - 1;
            if (ns < 2) {
              const uint4 *src = reinterpret_cast<const uint4 *>(ring_s2(ns, nl));
#pragma unroll
              for (int q = 0; q < 4; ++q) sq[q] = ld_global_v4_hint(src + (size_t)((col0 >> 3) + q) * 128 + row, pol_stream);
            }
          }
          if (l >= nu) {  // db of a fused layer: column sums of delta over the warp's 32 rows
            float d[32];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              d[2 * i] = bf16lo(dp[i]);
              d[2 * i + 1] = bf16hi(dp[i]);
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
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (j == l - nu) dbacc[j] += d[0];
          }
        }
        // the l = 0 step (dW MMA or delta_0 store) must retire before sA is rewritten
        mbar_wait_sleep(acc_full, accph);
        PH_MARK(5);
        accph ^= 1;
        tc_fence_after();
      }
    }
    // ------------------------------------------------------------ flush per-CTA partials
#ifdef DINR_PHASES
    if (tid == 0 && p.dbg)
      for (int k = 0; k < 8; ++k) p.dbg[(size_t)blockIdx.x * 8 + k] = ph[k];
#endif
    named_sync(1, EPI);
    for (int j = 0; j < nf; ++j) {
      uint32_t v[32];
      tmem_ld32(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(H + j * H + col0), v);
      tmem_wait_ld();
      if (H >= 128 || row < 64) {
        float *dst = p.dw_part + (((size_t)j * gridDim.x + blockIdx.x) * 128 + row) * H + col0;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          reinterpret_cast<float4 *>(dst)[q] = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                                           __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]));
      }
    }
    // db of fused layers: combine the 4 row-warps of each column group through smem
    float *red = sHsum;  // reuse: [4 row chunks][H + 4]
    for (int j = 0; j < nf; ++j) {
      named_sync(1, EPI);
      red[(warp & 3) * (H + 4) + col0 + lane] = dbacc[j];
      named_sync(1, EPI);
      if (tid < H) {
        float a = 0.f;
        for (int w = 0; w < 4; ++w) a += red[w * (H + 4) + tid];
        p.db_part[((size_t)j * gridDim.x + blockIdx.x) * 128 + tid] = a;
      }
    }
    named_sync(1, EPI);
    if ((warp & 3) == 0) p.head_part[(size_t)blockIdx.x * (H + 1) + col0 + lane] = wo_acc;
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
