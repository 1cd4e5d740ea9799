// k_tc_dwz.cuh -- weight-gradient GEMM of the H = 256 split path when the forward stashes only
// y_l = z_l / 2 (k_tc_fwd3 "zall"), part of north_star subsystem (3) (eq:partiald):
//   dW_l[o][i] = sum_samples delta_l[s][o] h_l[s][i]
// with the layer input h_l rebuilt on chip: layer 0 from the ray records (GRFF features, the
// forward's own arithmetic), layer l >= 1 as swish(z_{l-1}) = y (1 + tanh y) from the fp16 y stash.
// (db_l comes from K3's ones-MMA: this kernel's TMEM holds the whole 256 x 256 dW_l.)
//
// One CTA per (layer, K-split): both 128-row output blocks at once (M = 2 x 128, N = 256), so every
// h tile is built once (k_tc_dw's one-block CTAs would each rebuild it: twice the MUFU work).  The
// K loop runs over half tiles (64 samples): stage = delta^T [4 feature blocks][64 rows][128 B]
// (4 bulk copies of 8 KB) + h [4 feature blocks][64 rows][128 B] built by 16 converter warps
// (thread = sample row x 32-feature eighth: 32 tanh or 16 sin/cos pairs per half tile).  Every
// kDwFlushTiles tiles the same warps add the accumulator into the CTA's fp32 partial slot in
// global memory (read-modify-write of a slot only this CTA owns: deterministic; short fp32
// accumulation chains, see k_tc_dw.cuh).
#pragma once
#include "internal.cuh"
#include "k_features.cuh"
#include "k_tc_dw.cuh"
#include "ptx_sm100.cuh"

namespace dinr {

struct DwzLayout {
  static constexpr int H = 256;
  static constexpr uint32_t HALF = 4 * 8192;       // one operand of a half tile: 4 blocks x 64 rows x 128 B
  static constexpr uint32_t STAGE = 2 * HALF;      // delta^T + h
  static constexpr int NST = 3;
  static constexpr int NCONV = 16;                 // converter / flush warps (2 .. 17)
  static constexpr int NT = 64 + 32 * NCONV;       // warp 0: copies, warp 1: MMA
  static size_t smem_bytes() { return 1024 + (size_t)NST * STAGE + (H / 2) * 16 + 256; }
};

__global__ void __launch_bounds__(DwzLayout::NT, 1) k_tc_dwz(DwParams p) {
  using LY = DwzLayout;
  constexpr int H = LY::H, NST = LY::NST, C = H / 2;
  constexpr uint32_t HALF = LY::HALF;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float4 *sB4 = reinterpret_cast<float4 *>(smem + NST * LY::STAGE);
  uint64_t *full = reinterpret_cast<uint64_t *>(sB4 + H / 2);
  uint64_t *empty = full + NST;
  uint64_t *flush_full = empty + NST, *flush_free = flush_full + 1;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(flush_free + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int l = (int)blockIdx.x / p.ks1, split = (int)blockIdx.x % p.ks1, ks = p.ks1;
  if (warp == 0) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1 + LY::NCONV);  // the delta copies + one arrival per converter warp
      mbar_init(&empty[s], 1);
    }
    mbar_init(flush_full, 1);
    mbar_init(flush_free, LY::NCONV);
    fence_mbar_init();
  }
  for (int i = tid; i < H / 2; i += LY::NT) sB4[i] = reinterpret_cast<const float4 *>(p.B)[i];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  int count = 0;  // tiles of this CTA; the K loop has 2 count half tiles
  for (int64_t t = split; t < p.n_tiles; t += ks) ++count;
  const int nch = (count + kDwFlushTiles - 1) / kDwFlushTiles;

  if (tid == 0) {
    int it = 0;  // half-tile index
    for (int64_t t = split; t < p.n_tiles; t += ks)
      for (int hh = 0; hh < 2; ++hh, ++it) {
        const int st = it % NST;
        if (it >= NST) mbar_wait(&empty[st], ((it / NST) - 1) & 1);
        mbar_arrive_expect_tx(&full[st], HALF);
        const uint8_t *src = p.dstash + ((size_t)l * p.n_tiles + t) * (H * 256) + (size_t)hh * 8192;
        for (int fb = 0; fb < 4; ++fb) bulk_g2s(smem + st * LY::STAGE + fb * 8192, src + (size_t)fb * 16384, 8192, &full[st]);
      }
  } else if (tid == 32) {
    const uint32_t id_dw = idesc_bf16(128, H, 1, 1);
    for (int it = 0; it < 2 * count; ++it) {
      const int st = it % NST, ci = it % (2 * kDwFlushTiles);
      mbar_wait(&full[st], (it / NST) & 1);
      if (ci == 0 && it > 0) mbar_wait(flush_free, ((it / (2 * kDwFlushTiles)) - 1) & 1);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + st * LY::STAGE), sb = sa + HALF;
#pragma unroll
      for (int mb = 0; mb < 2; ++mb)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {  // K = 64 samples of the half tile, 16 per MMA
          const uint64_t ad = sdesc_sw128(sa + mb * 16384 + kk * 2048, 8192, 1024);
          const uint64_t bd = sdesc_sw128(sb + kk * 2048, 8192, 1024);
          umma_bf16(tmem + mb * 256, ad, bd, id_dw, (ci > 0 || kk > 0) ? 1u : 0u);
        }
      umma_commit(&empty[st]);
      if (ci == 2 * kDwFlushTiles - 1 || it == 2 * count - 1) umma_commit(flush_full);
    }
  } else if (warp >= 2) {
    // ============================================================ converters + flushes
    const int w = warp - 2;
    const int r = ((w & 1) << 5) | lane;  // sample row of the half tile (0..63)
    const int e8 = w >> 1;                 // features [32 e8, 32 e8 + 32) (layer >= 1); frequencies [16 e8, +16) (layer 0)
    // flush mapping: accumulator lane o (128) x 128-column quarter of the 512 (m-block = quarter / 2);
    // a warp may only read the TMEM lane quadrant warp % 4
    const int q4 = warp & 3, fq = w >> 2, o = (q4 << 5) | lane;
    const uint32_t trow = (uint32_t)(q4 * 32) << 16;
    float *dst = p.dw_part + ((((size_t)l * 2 + (fq >> 1)) * p.ksplit + split) * 128 + o) * H + (fq & 1) * 128;
    int c0 = 0;
    auto flush = [&](int c) {  // accumulator chunk c -> the CTA's partial slot
      mbar_wait(flush_full, c & 1);
      tc_fence_after();
#pragma unroll 1
      for (int h = 0; h < 4; ++h) {
        uint32_t v[32];
        tmem_ld32(tmem + trow + fq * 128 + h * 32, v);
        tmem_wait_ld();
        float4 *d4 = reinterpret_cast<float4 *>(dst + h * 32);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float4 a = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                                 __uint_as_float(v[4 * q + 3]));
          if (c > 0) {
            const float4 b = d4[q];
            a.x += b.x;
            a.y += b.y;
            a.z += b.z;
            a.w += b.w;
          }
          d4[q] = a;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(flush_free);
    };
    int it = 0;
    for (int64_t t = split; t < p.n_tiles; t += ks) {
      for (int hh = 0; hh < 2; ++hh, ++it) {
        // chunk c is flushed once its last half tile is NST behind (before the half tile whose
        // stage its restart holds back; see k_tc_dw.cuh)
        while (c0 < nch && 2 * (c0 + 1) * kDwFlushTiles - 1 <= it - NST) flush(c0++);
        const int st = it % NST;
        const uint32_t sb = smem_u32(smem + st * LY::STAGE + HALF);
        if (l == 0) {
          const int64_t g = t * 128 + hh * 64 + r;
          const float4 rb = grff_coords(p.rec32, g, p.lg_ns, p.n_s, g < p.nsamp, p.jit);
          if (it >= NST) mbar_wait(&empty[st], ((it / NST) - 1) & 1);
#pragma unroll
          for (int f0 = e8 * 16; f0 < e8 * 16 + 16; f0 += 8) {
            uint32_t pc[4], ps[4];
            grff8(sB4, f0, rb, pc, ps);
            st_shared_v4(sb + sw128_offset(r, f0, 64), pc[0], pc[1], pc[2], pc[3]);
            st_shared_v4(sb + sw128_offset(r, C + f0, 64), ps[0], ps[1], ps[2], ps[3]);
          }
        } else {
          // y chunks 2 e8, 2 e8 + 1 (16 features each) of row 64 hh + r
          const uint8_t *ysrc =
              p.ystash + ((((size_t)(l - 1) * p.n_tiles + t) * (H / 16) + 2 * e8) * 128 + hh * 64 + r) * 32;
          uint4 ya[2], yb[2];
#pragma unroll
          for (int c = 0; c < 2; ++c) ld_global_v8_hint(ysrc + (size_t)c * 128 * 32, ya[c], yb[c], policy_evict_first());
          if (it >= NST) mbar_wait(&empty[st], ((it / NST) - 1) & 1);
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const uint32_t yy[8] = {ya[c].x, ya[c].y, ya[c].z, ya[c].w, yb[c].x, yb[c].y, yb[c].z, yb[c].w};
            uint32_t w8[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float2 yf = __half22float2(*reinterpret_cast<const __half2 *>(&yy[e]));
#ifdef DINR_ZALL_F32_TANH
              w8[e] = pack_bf16x2(fmaf(yf.x, tanh_approx(yf.x), yf.x), fmaf(yf.y, tanh_approx(yf.y), yf.y));
#else  // one MUFU op for both (bf16x2 tanh: the h it feeds is rounded to bf16 right after)
              const uint32_t tt = bf2_tanh(pack_bf16x2(yf.x, yf.y));
              w8[e] = pack_bf16x2(fmaf(yf.x, bf16lo(tt), yf.x), fmaf(yf.y, bf16hi(tt), yf.y));
#endif
            }
            const int col = e8 * 32 + c * 16;
            st_shared_v4(sb + sw128_offset(r, col, 64), w8[0], w8[1], w8[2], w8[3]);
            st_shared_v4(sb + sw128_offset(r, col + 8, 64), w8[4], w8[5], w8[6], w8[7]);
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[st]);
      }
    }
    while (c0 < nch) flush(c0++);
    if (count == 0)  // nothing accumulated: the slot is zero
      for (int q = 0; q < 128; ++q) dst[q] = 0.f;
    // slots this layer does not use (ks < ksplit) are zero for the fixed-order reduction
    for (int s2 = split + ks; s2 < p.ksplit; s2 += ks) {
      float *z = p.dw_part + ((((size_t)l * 2 + (fq >> 1)) * p.ksplit + s2) * 128 + o) * H + (fq & 1) * 128;
      for (int q = 0; q < 128; ++q) z[q] = 0.f;
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
