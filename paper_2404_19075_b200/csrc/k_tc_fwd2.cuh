// k_tc_fwd2.cuh -- split-path training forward (K2, k_tc_mlp MODE 1) for H = 256 with two
// concurrent tile streams per CTA, north_star subsystem (2).
//
// k_tc_mlp runs one 128-sample tile per CTA: the tensor core idles during every epilogue, because
// the next layer's input is that epilogue's output.  Two tiles per CTA need two 64 KB A tiles; the
// full 128 KB W_l image does not fit beside them, so W_l is streamed as two 64 KB N-halves (output
// features [128 h, 128 h + 128)) that both streams consume before the buffer is refilled:
//   per layer: W_l half 0 -> MMA(s0, h0), MMA(s1, h0); W_l half 1 -> MMA(s0, h1), MMA(s1, h1)
// so stream 0's epilogue of layer l runs during stream 1's last MMA and the next weight load, and
// stream 1's during stream 0's next-layer MMAs.  Same math, rounding and outputs as k_tc_mlp
// MODE 1: ray-chunk sums of M, bulk stores of every layer input h_l (features for l = 0) to the
// h stash, 256-bit stores of swish'(z_l) (bf16, hidden layers) / z_{L-1} (fp16) to the s2 stash.
//   warps 0-7: stream 0 epilogue, warps 8-15: stream 1 (thread = sample row x column half)
//   warp 16 lane 0: weight loads, MMA issue, stash bulk stores
// TMEM: stream s accumulates in columns [256 s, 256 s + 256).
#pragma once
#include "internal.cuh"
#include "k_features.cuh"
#include "k_tc_mlp.cuh"
#include "ptx_sm100.cuh"

namespace dinr {

struct Fwd2Layout {
  static constexpr int H = 256, C = 128;
  static constexpr int NT = 512 + 32;
  static constexpr uint32_t A_BYTES = H * 256u;     // 128 rows x 256 bf16
  static constexpr uint32_t WH_BYTES = H * 256u;    // 128 output rows x 256 inputs
  static size_t smem_bytes(int L) {
    return 1024 + 2 * (size_t)A_BYTES + WH_BYTES + (size_t)L * H * 4 + (H + 4) * 4 + C * 16 + 2 * 2 * 128 * 4 + 256;
  }
};

__global__ void __launch_bounds__(Fwd2Layout::NT, 1) k_tc_fwd2(TcParams p) {
  using LY = Fwd2Layout;
  constexpr int H = LY::H, C = LY::C;
  constexpr uint32_t A_BYTES = LY::A_BYTES, W_LAYER = H * H * 2u;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared address space
  const int L = p.L;
  uint8_t *sA0 = smem;                                   // A tiles of streams 0, 1
  uint8_t *sW = sA0 + 2 * A_BYTES;                       // one W_l N-half image: [4 K-blocks][128 rows][128 B]
  float *sBias = reinterpret_cast<float *>(sW + LY::WH_BYTES);
  float *sWo = sBias + L * H;                            // w_o[H], b_o
  float *sB = sWo + H + 4;                               // C x 4
  float *sMu = sB + C * 4;                               // [2 streams][2 column halves][128 rows]
  uint64_t *bars = reinterpret_cast<uint64_t *>(sMu + 2 * 2 * 128);
  uint64_t *a_full = bars, *acc_full = bars + 2;         // [2] each
  uint64_t *w_bar = bars + 4, *w_free = bars + 5;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 6);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  if (tid == 512) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&a_full[s], 1);
      mbar_init(&acc_full[s], 2);  // MMA commit + the control thread once its stash store has read A_s
    }
    mbar_init(w_bar, 1);
    mbar_init(w_free, 1);
    fence_mbar_init();
  }
  const int64_t per = (int64_t)H * H + H;
  for (int i = tid; i < L * H; i += LY::NT) sBias[i] = p.params[(i / H) * per + (int64_t)H * H + (i % H)];
  for (int i = tid; i <= H; i += LY::NT) sWo[i] = p.params[(int64_t)L * per + i];
  for (int i = tid; i < C * 4; i += LY::NT) sB[i] = p.B[i];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t n_pairs = p.n_tiles / 2;  // the plan rounds the tile count up to even

  if (tid >= 512) {
    if (tid == 512) {
      // ============================================================ control: weights, MMA, stash
      const uint32_t a_base0 = smem_u32(sA0), w_base = smem_u32(sW);
      const uint32_t idesc = idesc_bf16(128, 128, 0, 0);
      const uint8_t *wsrc = reinterpret_cast<const uint8_t *>(p.wpack);
      uint32_t aph[2] = {0, 0}, wph = 0, fph = 0;
      bool first = true;
      for (int64_t pi = blockIdx.x; pi < n_pairs; pi += gridDim.x) {
        for (int l = 0; l < L; ++l) {
          for (int h = 0; h < 2; ++h) {
            // W_l output half h into the buffer once every MMA reading the previous half retired
            if (!first) {
              mbar_wait(w_free, fph);
              fph ^= 1;
            }
            first = false;
            mbar_arrive_expect_tx(w_bar, LY::WH_BYTES);
            for (int kb = 0; kb < 4; ++kb)
              bulk_g2s(sW + kb * 16384, wsrc + (size_t)l * W_LAYER + kb * (H * 128) + h * 16384, 16384, w_bar);
            {  // the next half into L2 meanwhile
              const int nl = h == 0 ? l : l + 1, nh = h ^ 1;
              if (nl < L)
                for (int kb = 0; kb < 4; ++kb)
                  bulk_prefetch_l2(wsrc + (size_t)nl * W_LAYER + kb * (H * 128) + nh * 16384, 16384);
            }
            mbar_wait(w_bar, wph);
            wph ^= 1;
            for (int s = 0; s < 2; ++s) {
              const int64_t tile = 2 * pi + s;
              const uint32_t a_base = a_base0 + s * A_BYTES;
              if (h == 0) {
                mbar_wait(&a_full[s], aph[s]);
                aph[s] ^= 1;
                // layer l's input for the dW GEMM (l = 0: the GRFF features; K5 reads the stash)
                if (l > 0 || p.stash_feat) {
                  bulk_s2g(p.hstash + ((size_t)l * p.n_tiles + tile) * A_BYTES, sA0 + s * A_BYTES, A_BYTES);
                  bulk_commit();
                }
              }
              tc_fence_after();
#pragma unroll 4
              for (int kk = 0; kk < H / 16; ++kk) {
                uint64_t ad = sdesc_sw128(a_base + (kk >> 2) * (128 * 128) + (kk & 3) * 32, 16, 1024);
                uint64_t bd = sdesc_sw128(w_base + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
                umma_bf16(tmem + s * 256 + h * 128, ad, bd, idesc, kk > 0 ? 1u : 0u);
              }
              if (h == 1) {
                umma_commit(&acc_full[s]);
                bulk_wait_read_all();  // the stash store of A_s has read it: the epilogue may overwrite
                mbar_arrive(&acc_full[s]);
              }
            }
            umma_commit(w_free);
          }
        }
      }
      bulk_wait_all();
    }
  } else {
    // ============================================================ epilogue streams
    const int s = tid >> 8, wt = tid & 255;
    const int row = wt & 127, cg = wt >> 7;
    const uint32_t a_base = smem_u32(sA0) + s * A_BYTES;
    const uint32_t tmem_row = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(s * 256);
    const uint64_t pol_z = policy_evict_first();
    uint32_t accph = 0;
    auto hand_off = [&]() {  // A_s written (generic proxy) -> the control thread's MMA / bulk reads
      fence_proxy_async_smem();
      asm volatile("bar.sync %0, 256;" ::"r"(1 + s) : "memory");
      if (wt == 0) mbar_arrive(&a_full[s]);
    };
    for (int64_t pi = blockIdx.x; pi < n_pairs; pi += gridDim.x) {
      const int64_t tile = 2 * pi + s;
      const int64_t g = tile * 128 + row;
      const bool valid = g < p.nsamp;
      // ---------------------------------------------------------------- a5/a6 features (as K2)
      {
        float rb0 = 0.f, rb1 = 0.f, rb2 = 0.f, rb3 = 0.f;
        if (valid) {
          int64_t ray = ray_of(g, p.n_s);
          const uint32_t jr = (uint32_t)(g - ray * p.n_s);
          float jj = (float)jr + sample_offset(p.jit, ray, jr);
          float4 ra = p.rec32[2 * ray], rbv = p.rec32[2 * ray + 1];
          rb0 = ra.w;
          rb1 = ra.z + jj * rbv.z;
          rb2 = ra.y + jj * rbv.y;
          rb3 = ra.x + jj * rbv.x;
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
              float fr = phi - rintf(phi);
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
      hand_off();
      // ---------------------------------------------------------------- a7/a8 layers
      float mu_acc = 0.f;
      for (int l = 0; l < L; ++l) {
        const bool last = (l == L - 1);
        mbar_wait(&acc_full[s], accph);
        accph ^= 1;
        tc_fence_after();
#pragma unroll 1
        for (int cb = cg * 4; cb < cg * 4 + 4; ++cb) {  // this thread's 32-column chunks
#pragma unroll
          for (int q16 = 0; q16 < 2; ++q16) {
            uint32_t v[16];
            tmem_ld16(tmem_row + cb * 32 + q16 * 16, v);
            tmem_wait_ld();
            const int col0 = cb * 32 + q16 * 16;
            float z[16], sg[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              z[i] = __uint_as_float(v[i]) + sBias[l * H + col0 + i];
              sg[i] = 0.5f + 0.5f * tanh_approx(0.5f * z[i]);
            }
            {  // backward state, [16-column chunk][row][32 B] (the layout K3 reads)
              uint32_t h8[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const int i0 = 2 * e;
                if (last) {
                  __half2 hh = __floats2half2_rn(z[i0], z[i0 + 1]);
                  h8[e] = *reinterpret_cast<uint32_t *>(&hh);
                } else {
                  h8[e] = pack_bf16x2(sg[i0] * (1.f + z[i0] * (1.f - sg[i0])), sg[i0 + 1] * (1.f + z[i0 + 1] * (1.f - sg[i0 + 1])));
                }
              }
              st_global_v8_hint(p.zstash + ((((size_t)l * p.n_tiles + tile) * (H / 16) + (col0 >> 4)) * 128 + row) * 32, h8,
                                pol_z);
            }
            if (!last) {
              uint32_t w8[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) w8[e] = pack_bf16x2(z[2 * e] * sg[2 * e], z[2 * e + 1] * sg[2 * e + 1]);
              st_shared_v4(a_base + sw128_offset(row, col0, 128), w8[0], w8[1], w8[2], w8[3]);
              st_shared_v4(a_base + sw128_offset(row, col0 + 8, 128), w8[4], w8[5], w8[6], w8[7]);
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i) mu_acc += sWo[col0 + i] * (z[i] * sg[i]);
            }
          }
        }
        tc_fence_before();
        if (!last) hand_off();
      }
      // a9 ray-chunk sum of M = mu0 (w_o . h_L + b_o) over each warp's 32 samples
      sMu[(s * 2 + cg) * 128 + row] = mu_acc;
      asm volatile("bar.sync %0, 256;" ::"r"(1 + s) : "memory");
      if (cg == 0) {
        float mu = p.mu0 * (sMu[(s * 2) * 128 + row] + sMu[(s * 2 + 1) * 128 + row] + sWo[H]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mu += __shfl_xor_sync(0xffffffffu, mu, o);
        if (lane == 0 && valid) p.pchunk[g >> 5] = mu;
      }
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
