// k_infer.cuh -- NEXT row N4: inference voxelization.
//
// Evaluates the trained field mu(x, y, z, t) = mu0 (w_o . h_L + b_o) (R6) at the voxel
// centres of a regular grid at one view time t, forward only.  Same MLP core as the fused
// training kernel (k_fused2.cuh): weights resident in shared memory as SW128 K-major images of
// W_l / 2, biases as one extra K = 16 MMA step, packed-bf16 Swish epilogue; two 128-voxel tile
// streams per CTA on two epilogue warpgroups so the tensor core works on one stream's layer
// while the other stream's epilogue runs.  No reductions: every voxel writes one fp32 value.
// Voxels outside the FOV cylinder (x - x_s0)^2 + y^2 <= r^2 are 0 (R25; decided in fp64).
#pragma once
#include "internal.cuh"
#include "k_features.cuh"
#include "ptx_sm100.cuh"

namespace dinr {

struct InferParams {
  VoxGrid vg;
  int64_t n_vox;  // voxels in this launch (slab of whole z planes)
  int L;
  float mu0;
  const float *params;
  const float *B;
  const uint16_t *wpack_half;  // L x W_l / 2 images (SW128 K-major)
  float *out;
};

template <int H>
struct InferLayout {
  static constexpr int EPI = 512;
  static constexpr int NT = EPI + 32;
  static constexpr uint32_t TILE = H * 256u;
  static constexpr uint32_t A_BYTES = H == 64 ? 2 * TILE : TILE;  // H = 64: K = 64 uses one 128-B block
  static constexpr uint32_t W_LAYER = H * H * 2u;
  static constexpr uint32_t ONES = 128 * 32;
  static constexpr uint32_t BIAS_B = H * 32;
  static size_t smem_bytes(int L) {
    return 1024 + 2 * (size_t)A_BYTES + (size_t)L * W_LAYER + ONES + (size_t)L * BIAS_B + (H + 4) * 4 + (H / 2) * 16 +
           2 * 128 * 2 * 4 + 128;
  }
};

template <int H>
__global__ void __launch_bounds__(InferLayout<H>::NT, 1) k_infer(InferParams p) {
  using LY = InferLayout<H>;
  constexpr int C = H / 2;
  constexpr int EPI = LY::EPI;
  constexpr uint32_t TILE = LY::TILE;
  constexpr int NHC = H / 32;  // 16-column steps per thread (column half of H)
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int L = p.L;
  uint8_t *sA0 = smem;
  uint8_t *sW = sA0 + 2 * LY::A_BYTES;
  uint8_t *sOnes = sW + (size_t)L * LY::W_LAYER;
  uint8_t *sBiasB = sOnes + LY::ONES;
  float *sWo = reinterpret_cast<float *>(sBiasB + (size_t)L * LY::BIAS_B);  // w_o[H], b_o
  float *sB = sWo + H + 4;                                                   // C x 4
  float *sMu = sB + C * 4;                                                   // [2 streams][128 rows][2 halves]
  uint64_t *bars = reinterpret_cast<uint64_t *>(sMu + 2 * 128 * 2);
  uint64_t *a_full = bars, *acc_full = bars + 2, *w_bar = bars + 4;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 5);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    tmem_alloc(tmem_slot, 2 * H);
    tmem_relinquish();
  }
  if (tid == EPI) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&a_full[s], 8);
      mbar_init(&acc_full[s], 1);
    }
    mbar_init(w_bar, 1);
    fence_mbar_init();
  }
  const int64_t per = (int64_t)H * H + H;
  for (int i = tid; i < (int)(LY::ONES + L * LY::BIAS_B) / 4; i += LY::NT) reinterpret_cast<uint32_t *>(sOnes)[i] = 0u;
  if (H == 64)
    for (int i = tid; i < (int)(2 * TILE / 16); i += LY::NT) {
      const int s = i / (TILE / 16), k = i % (TILE / 16);
      reinterpret_cast<uint4 *>(sA0 + s * LY::A_BYTES + TILE)[k] = make_uint4(0, 0, 0, 0);
    }
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
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t a0_base = smem_u32(sA0), w_base = smem_u32(sW);
  const uint32_t ones_base = smem_u32(sOnes), biasb_base = smem_u32(sBiasB);
  const int64_t n_groups = (p.n_vox + 255) / 256;

  if (tid >= EPI) {
    // ===================================================== MMA issuer
    if (lane == 0) {
      const uint32_t idf = idesc_bf16(128, H, 0, 0);
      const uint32_t wb = (uint32_t)L * LY::W_LAYER;
      mbar_arrive_expect_tx(w_bar, wb);
      for (uint32_t off = 0; off < wb; off += 32768u)
        bulk_g2s(sW + off, reinterpret_cast<const uint8_t *>(p.wpack_half) + off, min(32768u, wb - off), w_bar);
      mbar_wait(w_bar, 0);
      uint32_t aph[2] = {0, 0};
      for (int64_t gi = blockIdx.x; gi < n_groups; gi += gridDim.x)
        for (int l = 0; l < L; ++l)
          for (int s = 0; s < 2; ++s) {
            const uint32_t a_base = a0_base + s * LY::A_BYTES;
            mbar_wait(&a_full[s], aph[s]);
            aph[s] ^= 1;
            tc_fence_after();
            const uint32_t wl = w_base + (uint32_t)l * LY::W_LAYER;
            umma_bf16(tmem + s * H, sdesc_none(ones_base, 128, 256), sdesc_none(biasb_base + l * LY::BIAS_B, 128, 256),
                      idf, 0u);
#pragma unroll
            for (int kk = 0; kk < H / 16; ++kk)
              umma_bf16(tmem + s * H, sdesc_sw128(a_base + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                        sdesc_sw128(wl + (kk >> 2) * (H * 128) + (kk & 3) * 32, 16, 1024), idf, 1u);
            umma_commit(&acc_full[s]);
          }
    }
    __syncwarp();
  } else {
    // ===================================================== epilogue warpgroups
    const int s = tid >> 8, wt = tid & 255;
    const int row = wt & 127, ch = wt >> 7;
    const uint32_t a_base = a0_base + s * LY::A_BYTES;
    const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(s * H + ch * (H / 2));
    uint32_t accph = 0;
    for (int64_t gi = blockIdx.x; gi < n_groups; gi += gridDim.x) {
      const int64_t v = (2 * gi + s) * 128 + row;
      const bool valid = v < p.n_vox;
      bool inside = false;
      const float4 rb = voxel_coords(p.vg, valid ? v : 0, inside);
      // features of this thread's half of the frequencies; A_s is free once the previous
      // group's last MMA has completed (waited below)
      constexpr int NFC = (C / 2) / 8;
#pragma unroll
      for (int fc = 0; fc < NFC; ++fc) {
        uint32_t pc[4], ps[4];
        const int c0 = ch * (C / 2) + 8 * fc;
        grff8(reinterpret_cast<const float4 *>(sB), c0, rb, pc, ps);
        st_shared_v4(a_base + sw128_offset(row, c0, 128), pc[0], pc[1], pc[2], pc[3]);
        st_shared_v4(a_base + sw128_offset(row, C + c0, 128), ps[0], ps[1], ps[2], ps[3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&a_full[s]);
      float mu_part = 0.f;
      for (int l = 0; l < L; ++l) {
        const bool last = l == L - 1;
        mbar_wait(&acc_full[s], accph);
        accph ^= 1;
        tc_fence_after();
#pragma unroll
        for (int hc = 0; hc < NHC; ++hc) {
          uint32_t cur[16];
          tmem_ld16(trow + hc * 16, cur);
          tmem_wait_ld();
          const int col0 = ch * (H / 2) + hc * 16;
          uint32_t hpk[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint32_t yb = pack_bf16x2(__uint_as_float(cur[2 * i]), __uint_as_float(cur[2 * i + 1]));
            hpk[i] = bf2_fma(yb, bf2_tanh(yb), yb);  // swish(z) = y (1 + tanh y), y = z / 2
          }
          if (!last) {
#pragma unroll
            for (int q = 0; q < 2; ++q)
              st_shared_v4(a_base + sw128_offset(row, col0 + 8 * q, 128), hpk[4 * q], hpk[4 * q + 1], hpk[4 * q + 2],
                           hpk[4 * q + 3]);
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              mu_part = fmaf(sWo[col0 + 2 * i], bf16lo(hpk[i]), mu_part);
              mu_part = fmaf(sWo[col0 + 2 * i + 1], bf16hi(hpk[i]), mu_part);
            }
          }
        }
        tc_fence_before();
        if (!last) {
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&a_full[s]);
        }
      }
      // a9 (per voxel): mu = mu0 (w_o . h_L + b_o); the two column halves of a row meet in smem
      sMu[(s * 128 + row) * 2 + ch] = mu_part;
      named_sync(1 + s, 256);
      if (ch == 0 && valid)
        p.out[v] = inside ? p.mu0 * (sMu[(s * 128 + row) * 2] + sMu[(s * 128 + row) * 2 + 1] + sWo[H]) : 0.f;
      named_sync(1 + s, 256);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 2 * H);
  }
}

}  // namespace dinr
