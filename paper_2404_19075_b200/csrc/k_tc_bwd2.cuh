// k_tc_bwd2.cuh -- split-path backward dX chain (K3, k_tc_mlp MODE 2) for H = 256 with two
// concurrent tile streams per CTA, north_star subsystem (3) (eq:partiald).
//
// k_tc_mlp MODE 2 runs one tile per CTA and streams the whole 128 KB W_l image per layer through
// one buffer: the tensor core idles during every weight load and every epilogue.  Here, as in the
// forward k_tc_fwd2, two tiles share each W_l load, streamed as two 64 KB halves of its MN-major
// dX operand (input features [128 h, 128 h + 128) = two contiguous 64-column blocks):
//   per layer l = L-1 .. 1: W_l half 0 -> MMA(s0, h0), MMA(s1, h0); half 1 -> MMA(s0, h1), MMA(s1, h1)
// so one stream's epilogue overlaps the other stream's MMAs and the next weight half's load.
// Same math, rounding and outputs as k_tc_mlp MODE 2: the top layer's delta and head gradients
// from the stashed fp16 z_{L-1} and the upstream u, then delta_{l-1} = (delta_l W_l) (.)
// swish'(z_{l-1}) (bf16 swish' from the forward's stash), every delta_l image bulk-stored to the
// delta stash for the dW GEMM (k_tc_dw.cuh).
//   warps 0-7: stream 0 epilogue, warps 8-15: stream 1 (thread = sample row x column half)
//   warp 16 lane 0: weight loads, MMA issue, delta-stash bulk stores
// TMEM: stream s accumulates e_{l-1} in columns [256 s, 256 s + 256).
#pragma once
#include "internal.cuh"
#include "k_tc_mlp.cuh"
#include "ptx_sm100.cuh"

namespace dinr {

struct Bwd2Layout {
  static constexpr int H = 256;
  static constexpr int NT = 512 + 32;
  static constexpr uint32_t A_BYTES = H * 256u;   // 128 rows x 256 bf16
  static constexpr uint32_t WH_BYTES = H * 256u;  // 256 output rows x 128 inputs (two 64-column blocks)
  static size_t smem_bytes() { return 1024 + 2 * (size_t)A_BYTES + WH_BYTES + (H + 4) * 4 + 256; }
};

__global__ void __launch_bounds__(Bwd2Layout::NT, 1) k_tc_bwd2(TcParams p, int nhead_slots) {
  using LY = Bwd2Layout;
  constexpr int H = LY::H;
  constexpr uint32_t A_BYTES = LY::A_BYTES, W_LAYER = H * H * 2u;
  constexpr int NCB = H / 64;                  // 32-column chunks of a thread's column half
  constexpr uint32_t kZTile = 128u * H * 2u;   // one tile of the 16-bit backward state
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared address space
  const int L = p.L;
  uint8_t *sA0 = smem;                                  // A tiles (delta_l images) of streams 0, 1
  uint8_t *sW = sA0 + 2 * A_BYTES;                      // one W_l half: [2 input blocks][256 rows][128 B]
  float *sWo = reinterpret_cast<float *>(sW + LY::WH_BYTES);  // w_o[H], b_o
  uint64_t *bars = reinterpret_cast<uint64_t *>(sWo + H + 4);
  uint64_t *a_full = bars, *acc_full = bars + 2;        // [2] each
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
      // A_s free / accumulator ready: the MMA commit + the control thread once its stash store has
      // read A_s (after the last delta_0 store, which no MMA follows, the control thread arrives twice)
      mbar_init(&acc_full[s], 2);
    }
    mbar_init(w_bar, 1);
    mbar_init(w_free, 1);
    fence_mbar_init();
  }
  const int64_t per = (int64_t)H * H + H;
  for (int i = tid; i <= H; i += LY::NT) sWo[i] = p.params[(int64_t)L * per + i];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t n_pairs = p.n_tiles / 2;  // the plan rounds the tile count up to even

  float head_acc[2 * NCB];  // per 16-column chunk of the thread's half: lanes l, l ^ 16 hold column l & 15
#pragma unroll
  for (int i = 0; i < 2 * NCB; ++i) head_acc[i] = 0.f;
  float bo_acc = 0.f;

  if (tid >= 512) {
    if (tid == 512) {
      // ============================================================ control: weights, MMA, stash
      const uint32_t a_base0 = smem_u32(sA0), w_base = smem_u32(sW);
      const uint32_t idesc = idesc_bf16(128, 128, 0, 1);  // A K-major (delta rows), B MN-major (W_l)
      const uint8_t *wsrc = reinterpret_cast<const uint8_t *>(p.wpack);
      uint32_t aph[2] = {0, 0}, wph = 0, fph = 0;
      bool first = true;
      for (int64_t pi = blockIdx.x; pi < n_pairs; pi += gridDim.x) {
        for (int l = L - 1; l >= 0; --l) {
          if (l == 0) {  // delta_0: stash it, no MMA follows
            for (int s = 0; s < 2; ++s) {
              mbar_wait(&a_full[s], aph[s]);
              aph[s] ^= 1;
              bulk_s2g(p.dstash + ((size_t)0 * p.n_tiles + 2 * pi + s) * A_BYTES, sA0 + s * A_BYTES, A_BYTES);
              bulk_commit();
            }
            for (int s = 0; s < 2; ++s) {
              bulk_wait_read_all();
              mbar_arrive(&acc_full[s]);
              mbar_arrive(&acc_full[s]);
            }
            continue;
          }
          for (int h = 0; h < 2; ++h) {
            // W_l input half h into the buffer once every MMA reading the previous half retired
            if (!first) {
              mbar_wait(w_free, fph);
              fph ^= 1;
            }
            first = false;
            mbar_arrive_expect_tx(w_bar, LY::WH_BYTES);
            bulk_g2s(sW, wsrc + (size_t)l * W_LAYER + (size_t)h * LY::WH_BYTES, 32768, w_bar);
            bulk_g2s(sW + 32768, wsrc + (size_t)l * W_LAYER + (size_t)h * LY::WH_BYTES + 32768, 32768, w_bar);
            {  // the next half into L2 meanwhile
              const int nl = h == 0 ? l : l - 1, nh = h ^ 1;
              if (nl >= 1) bulk_prefetch_l2(wsrc + (size_t)nl * W_LAYER + (size_t)nh * LY::WH_BYTES, LY::WH_BYTES);
            }
            mbar_wait(w_bar, wph);
            wph ^= 1;
            for (int s = 0; s < 2; ++s) {
              const int64_t tile = 2 * pi + s;
              const uint32_t a_base = a_base0 + s * A_BYTES;
              if (h == 0) {
                mbar_wait(&a_full[s], aph[s]);
                aph[s] ^= 1;
                // delta_l for the dW GEMM
                bulk_s2g(p.dstash + ((size_t)l * p.n_tiles + tile) * A_BYTES, sA0 + s * A_BYTES, A_BYTES);
                bulk_commit();
              }
              tc_fence_after();
#pragma unroll 4
              for (int kk = 0; kk < H / 16; ++kk) {  // K = the layer's output features (16 rows of W_l)
                uint64_t ad = sdesc_sw128(a_base + (kk >> 2) * (128 * 128) + (kk & 3) * 32, 16, 1024);
                uint64_t bd = sdesc_sw128(w_base + kk * 2048, H * 128, 1024);
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
    const int cb_lo = cg * NCB;
    const uint32_t a_base = smem_u32(sA0) + s * A_BYTES;
    const uint32_t tmem_row = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(s * 256);
    const uint64_t pol_z = policy_evict_first();
    uint32_t accph = 0;
    bool a_busy = false;  // A_s still read by the previous pair's last stash store
    auto hand_off = [&]() {  // A_s written (generic proxy) -> the control thread's MMA / bulk reads
      fence_proxy_async_smem();
      asm volatile("bar.sync %0, 256;" ::"r"(1 + s) : "memory");
      if (wt == 0) mbar_arrive(&a_full[s]);
    };
    for (int64_t pi = blockIdx.x; pi < n_pairs; pi += gridDim.x) {
      const int64_t tile = 2 * pi + s;
      const int64_t g = tile * 128 + row;
      const bool valid = g < p.nsamp;
      // ---------------------------------------------------------------- top layer (as K3)
      // (16-column steps: a 544-thread CTA has 96 registers per thread)
      const float u_row = valid ? p.u[ray_of(g, p.n_s)] : 0.f;
      {
        const uint8_t *zsrc = p.zstash + (((size_t)(L - 1) * p.n_tiles + tile) * (H / 16) * 128 + row) * 32;
        uint4 zt[2][2];  // this 16-column step's fp16 z and the next one's, in flight
        ld_global_v8_hint(zsrc + (size_t)(cb_lo * 2) * 128 * 32, zt[0][0], zt[0][1], pol_z);
        if (a_busy) {  // the previous pair's delta_0 store has read A_s
          mbar_wait(&acc_full[s], accph);
          accph ^= 1;
        }
        a_busy = true;
#pragma unroll
        for (int k = 0; k < 2 * NCB; ++k) {
          const int c16 = cb_lo * 2 + k;  // 16-column chunk
          if (k + 1 < 2 * NCB)
            ld_global_v8_hint(zsrc + (size_t)(c16 + 1) * 128 * 32, zt[(k + 1) & 1][0], zt[(k + 1) & 1][1], pol_z);
          float z[16];
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const uint4 zq4 = zt[k & 1][q];
            const uint32_t zz[4] = {zq4.x, zq4.y, zq4.z, zq4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 zf = __half22float2(*reinterpret_cast<const __half2 *>(&zz[e]));
              z[8 * q + 2 * e] = zf.x;
              z[8 * q + 2 * e + 1] = zf.y;
            }
          }
          float x[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) x[i] = u_row * swish_f(z[i]);
#pragma unroll
          for (int o = 8; o >= 1; o >>= 1) {  // column sums of u h_L over the warp's 32 rows
            const bool upper = (lane & o) != 0;
#pragma unroll
            for (int i = 0; i < o; ++i) {
              float send = upper ? x[i] : x[i + o];
              float keep = upper ? x[i + o] : x[i];
              x[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
          }
          x[0] += __shfl_xor_sync(0xffffffffu, x[0], 16);  // lanes l, l ^ 16: column l & 15
          head_acc[k] += x[0];
          uint32_t w8[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int i0 = 2 * e;
            const float d0 = u_row * sWo[c16 * 16 + i0] * dswish_f(z[i0]);
            const float d1 = u_row * sWo[c16 * 16 + i0 + 1] * dswish_f(z[i0 + 1]);
            w8[e] = pack_bf16x2(d0, d1);
          }
          st_shared_v4(a_base + sw128_offset(row, c16 * 16, 128), w8[0], w8[1], w8[2], w8[3]);
          st_shared_v4(a_base + sw128_offset(row, c16 * 16 + 8, 128), w8[4], w8[5], w8[6], w8[7]);
        }
        if (cg == 0) {
          float us = u_row;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) us += __shfl_xor_sync(0xffffffffu, us, o);
          bo_acc += us;
        }
        tc_fence_before();
        hand_off();
      }
      // ---------------------------------------------------------------- dX chain
      for (int l = L - 1; l >= 1; --l) {
        // swish'(z_{l-1}): the first half of this thread's 16-column chunks in flight while the dX
        // MMA runs, each of the others issued as a chunk is consumed (register budget)
        const uint8_t *zsrc = p.zstash + (((size_t)(l - 1) * p.n_tiles + tile) * (H / 16) * 128 + row) * 32;
        uint4 zq[2 * NCB][2];
#pragma unroll
        for (int k = 0; k < NCB; ++k) ld_global_v8_hint(zsrc + (size_t)(cb_lo * 2 + k) * 128 * 32, zq[k][0], zq[k][1], pol_z);
        if (l >= 2 && cg == 0 && (row & 31) == 0)  // the next step's state into L2 meanwhile
          bulk_prefetch_l2(p.zstash + ((size_t)(l - 2) * p.n_tiles + tile) * kZTile + (size_t)(row >> 5) * (kZTile / 4),
                           kZTile / 4);
        mbar_wait(&acc_full[s], accph);
        accph ^= 1;
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < 2 * NCB; ++k) {
          const int c16 = cb_lo * 2 + k;
          uint32_t v[16];
          tmem_ld16(tmem_row + c16 * 16, v);
          tmem_wait_ld();
          uint32_t w8[8];
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const uint32_t zz[4] = {zq[k][q].x, zq[k][q].y, zq[k][q].z, zq[k][q].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {  // delta = e swish'(z), swish' stashed as bf16 by the forward
              const int i0 = 8 * q + 2 * e;
              w8[4 * q + e] = pack_bf16x2(__uint_as_float(v[i0]) * bf16lo(zz[e]), __uint_as_float(v[i0 + 1]) * bf16hi(zz[e]));
            }
          }
          st_shared_v4(a_base + sw128_offset(row, c16 * 16, 128), w8[0], w8[1], w8[2], w8[3]);
          st_shared_v4(a_base + sw128_offset(row, c16 * 16 + 8, 128), w8[4], w8[5], w8[6], w8[7]);
          if (k + NCB < 2 * NCB)  // NCB chunks ahead, into the registers chunk k just released
            ld_global_v8_hint(zsrc + (size_t)(c16 + NCB) * 128 * 32, zq[k + NCB][0], zq[k + NCB][1], pol_z);
        }
        tc_fence_before();
        hand_off();
      }
    }
    if (a_busy) {  // the last delta_0 store has read A_s
      mbar_wait(&acc_full[s], accph);
      accph ^= 1;
    }
  }
  // ------------------------------------------------------------ per-CTA head partials
  __syncthreads();
  float *red = reinterpret_cast<float *>(sA0);  // both A tiles are free now
  if (tid < 512) {
    const int s = tid >> 8, wt = tid & 255, cg = wt >> 7, w8 = wt >> 5;  // w8: warp within the stream
    if (lane < 16)
#pragma unroll
      for (int k = 0; k < 2 * NCB; ++k) red[(s * 8 + w8) * (H + 1) + (cg * NCB * 2 + k) * 16 + lane] = head_acc[k];
    if (lane == 0) red[(s * 8 + w8) * (H + 1) + H] = bo_acc;  // (zero for column-half-1 warps)
  }
  __syncthreads();
  for (int k = tid; k <= H; k += LY::NT) {
    float acc = 0.f;
    const int w0 = (k < H && k >= H / 2) ? 4 : 0;  // the 4 warps of each stream's column half holding k
    for (int s = 0; s < 2; ++s)
      for (int w = w0; w < w0 + 4; ++w) acc += red[(s * 8 + w) * (H + 1) + k];
    p.head_part[(size_t)blockIdx.x * (H + 1) + k] = acc;
    for (int b = blockIdx.x + gridDim.x; b < nhead_slots; b += gridDim.x) p.head_part[(size_t)b * (H + 1) + k] = 0.f;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace dinr
