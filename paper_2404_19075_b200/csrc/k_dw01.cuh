// k_dw01.cuh -- weight gradients of layers 0 and 1 after the fused kernel (fan512 path, nu = 2),
// with both layer inputs and delta_0 recomputed on chip instead of stashed in HBM:
//   dW_0 = sum delta_0^T gamma(x),      db_0 = sum delta_0          (eq:partiald)
//   dW_1 = sum delta_1^T h_0,           db_1 = sum delta_1,    h_0 = swish(W_0 gamma(x) + b_0)
//   delta_0 = (delta_1 W_1) swish'(z_0)                             (the chain rule's last dX step)
// Everything is recomputed with the fused kernel's own code and rounding, so it equals, bit for
// bit, what that kernel would have formed: gamma(x) from the ray records (k_features.cuh), h_0 and
// s2_0 = 2 swish'(z_0) from one forward MMA with the same 0.5-prescaled bf16 W_0 image, bias MMA
// step and packed-bf16 Swish, e_0 = delta_1 W_1 / 2 by the same dX MMA.  Only delta_1 comes from HBM.
//   warp 0: bulk loads (W_0, W_1 once; delta_1 per tile, the next tile prefetched into L2);
//   warp 1: MMA issuer, per tile t: e_0(t), dW_1(t), y(t+1), dW_0(t);
//   warps 2-9: thread = (TMEM lane / sample row, column half): y -> h_0 tile and s2_0 (registers),
//              then e_0 -> delta_0 tile, both through the one HD tile buffer;
//   warps 10-17: thread = (sample row, frequency half): gamma(x) of the next tile -> F (2 buffers).
// TMEM: R [0, H) = y(t), then e_0(t); dW_0 [H, 2H), dW_1 [2H, 3H), db_0 / db_1 at 3H / 3H + 16.
#pragma once
#include "internal.cuh"
#include "k_features.cuh"
#include "ptx_sm100.cuh"

namespace dinr {

// waits spin by default (suspended try_waits overslept: +0.19 ms per step on fan512)
#ifdef DINR_DW01_SLEEP
#define DW01_WAIT(bar, ph) mbar_wait_sleep(bar, ph, 1000)
#else
#define DW01_WAIT(bar, ph) mbar_wait(bar, ph)
#endif

struct Dw01Params {
  const uint8_t *dstash;  // [nu][n_tiles] SW128 images of delta_l (only l = 1 is read)
  int64_t n_tiles, nsamp;
  const float4 *rec32;
  Jitter jit;
  const float *B;
  int n_s, lg_ns;
  const float *params;
  const uint16_t *wpack_half;  // W_0 / 2 image, then W_1 / 2
  float *dw_part, *db_part;    // [l][ksplit][128][H], [l][ksplit][128]; ksplit = gridDim.x
};

template <int H>
struct Dw01Layout {
  static constexpr int NQ = 2;             // column parts per sample row (Swish warps)
  static constexpr int NFW = 4 * NQ;       // Swish warps
  static constexpr int NFE = 8;            // GRFF feature warps
  static constexpr int NT = 64 + 32 * (NFW + NFE);
  static constexpr uint32_t TILE = H * 256u;
  static constexpr uint32_t ONES_K = 128 * 32;  // no-swizzle [128][16]: columns 0, 1 = 1 (bias MMA)
  static constexpr uint32_t BIAS_B = H * 32;
  static constexpr uint32_t ONES_N = 2048;      // SW128 K-major [16 rows][64] of ones (db MMA B operand)
  // delta_1, F x 2, HD (h_0 then delta_0), W_0, W_1
  static size_t smem_bytes() { return 1024 + 4 * (size_t)TILE + 2 * (size_t)H * H * 2 + ONES_K + BIAS_B + ONES_N + (H / 2) * 16 + 256; }
};

template <int H>
__global__ void __launch_bounds__(Dw01Layout<H>::NT, 1) k_dw01(Dw01Params p) {
  static_assert(H == 128, "k_dw01 is the H = 128 path");
  using LY = Dw01Layout<H>;
  constexpr int C = H / 2;
  constexpr uint32_t TILE = LY::TILE;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *sD1 = smem;                         // delta_1 tile
  uint8_t *sF = sD1 + TILE;                    // gamma(x) tiles (double-buffered)
  uint8_t *sHD = sF + 2 * TILE;                // h_0 tile, then delta_0 tile
  uint8_t *sW0 = sHD + TILE;                   // W_0 / 2
  uint8_t *sW1 = sW0 + (size_t)H * H * 2;      // W_1 / 2
  uint8_t *sOnesK = sW1 + (size_t)H * H * 2;
  uint8_t *sBias = sOnesK + LY::ONES_K;
  uint8_t *sOnesN = sBias + LY::BIAS_B;
  float4 *sB4 = reinterpret_cast<float4 *>(sOnesN + LY::ONES_N);
  uint64_t *bars = reinterpret_cast<uint64_t *>(sB4 + C);
  //   d1_full (tx)      delta_1(t) landed        d1_free (commit)  e_0(t), dW_1(t) read it
  //   fbar[b] (NFE)     F(t) in slot b = t % 2   f_free[b] (commit) y(t), dW_0(t) read F slot b
  //   y_full (commit)   y(t) in R                y_free (NFW)      Swish loaded y(t): e_0(t) may overwrite R
  //   e_full (commit)   e_0(t) in R              e_free (NFW)      e_0(t) loaded: y(t+1) may overwrite R
  //   h_full (NFW)      h_0(t) in HD             h_done (commit)   dW_1(t) read h_0(t): delta_0(t) may overwrite
  //   d0_full (NFW)     delta_0(t) in HD         d0_done (commit)  dW_0(t) read delta_0(t): h_0(t+1) may overwrite
  uint64_t *d1_full = bars, *d1_free = bars + 1, *fbar = bars + 2, *f_free = bars + 4;
  uint64_t *y_full = bars + 6, *y_free = bars + 7, *e_full = bars + 8, *e_free = bars + 9;
  uint64_t *h_full = bars + 10, *h_done = bars + 11, *d0_full = bars + 12, *d0_done = bars + 13;
  uint64_t *w_bar = bars + 14, *done = bars + 15;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 16);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  if (tid == 0) {
    mbar_init(d1_full, 1);
    mbar_init(d1_free, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&fbar[b], LY::NFE);
      mbar_init(&f_free[b], 1);
    }
    mbar_init(y_full, 1);
    mbar_init(y_free, LY::NFW);
    mbar_init(e_full, 1);
    mbar_init(e_free, LY::NFW);
    mbar_init(h_full, LY::NFW);
    mbar_init(h_done, 1);
    mbar_init(d0_full, LY::NFW);
    mbar_init(d0_done, 1);
    mbar_init(w_bar, 1);
    mbar_init(done, 1);
    fence_mbar_init();
  }
  for (int i = tid; i < (int)(LY::ONES_K + LY::BIAS_B) / 4; i += LY::NT) reinterpret_cast<uint32_t *>(sOnesK)[i] = 0u;
  for (int i = tid; i < (int)LY::ONES_N / 4; i += LY::NT) reinterpret_cast<uint32_t *>(sOnesN)[i] = 0x3F803F80u;
  for (int i = tid; i < C; i += LY::NT) sB4[i] = reinterpret_cast<const float4 *>(p.B)[i];
  __syncthreads();
  for (int i = tid; i < 128; i += LY::NT) {
    *reinterpret_cast<__nv_bfloat16 *>(sOnesK + nosw16_offset(i, 0)) = __float2bfloat16_rn(1.f);
    *reinterpret_cast<__nv_bfloat16 *>(sOnesK + nosw16_offset(i, 1)) = __float2bfloat16_rn(1.f);
  }
  for (int i = tid; i < H; i += LY::NT) {  // b_0 / 2 as hi + lo (same split as the fused kernel)
    const float hb = 0.5f * p.params[(int64_t)H * H + i];
    const __nv_bfloat16 hi = __float2bfloat16_rn(hb);
    const __nv_bfloat16 lo = __float2bfloat16_rn(hb - __bfloat162float(hi));
    *reinterpret_cast<__nv_bfloat16 *>(sBias + nosw16_offset(i, 0)) = hi;
    *reinterpret_cast<__nv_bfloat16 *>(sBias + nosw16_offset(i, 1)) = lo;
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_r = tmem, t_dw0 = tmem + H, t_dw1 = tmem + 2 * H, t_db0 = tmem + 3 * H, t_db1 = tmem + 3 * H + 16;
  const int ks = gridDim.x, split = blockIdx.x;
  int count = 0;
  for (int64_t t = split; t < p.n_tiles; t += ks) ++count;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------- bulk loads
      mbar_arrive_expect_tx(w_bar, 2 * H * H * 2);
      bulk_g2s(sW0, p.wpack_half, H * H * 2, w_bar);
      bulk_g2s(sW1, p.wpack_half + H * H, H * H * 2, w_bar);
      const uint8_t *d1src = p.dstash + (size_t)p.n_tiles * TILE;  // layer 1's images
      int it = 0;
      for (int64_t t = split; t < p.n_tiles; t += ks, ++it) {
        if (t + ks < p.n_tiles) bulk_prefetch_l2(d1src + (size_t)(t + ks) * TILE, TILE);
        if (it >= 1) DW01_WAIT(d1_free, (it - 1) & 1);
        mbar_arrive_expect_tx(d1_full, TILE);
        bulk_g2s(sD1, d1src + (size_t)t * TILE, TILE, d1_full);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------- MMA issuer
      const uint32_t idf = idesc_bf16(128, H, 0, 0), idx = idesc_bf16(128, H, 0, 1), idw = idesc_bf16(128, H, 1, 1);
      const uint32_t idb = idesc_bf16(128, 16, 1, 0);
      const uint32_t f_base = smem_u32(sF), hd = smem_u32(sHD), d1 = smem_u32(sD1), on = smem_u32(sOnesN);
      const uint32_t w0 = smem_u32(sW0), w1 = smem_u32(sW1);
      mbar_wait(w_bar, 0);
      auto y_mma = [&](int it) {  // y(t) = gamma(x) W_0^T / 2 + b_0 / 2 into R
        const uint32_t fbase = f_base + (it & 1) * TILE;
        mbar_wait(&fbar[it & 1], (it >> 1) & 1);
        if (it > 0) mbar_wait(e_free, (it - 1) & 1);  // e_0(t-1) has been loaded from R
        tc_fence_after();
        umma_bf16(t_r, sdesc_none(smem_u32(sOnesK), 128, 256), sdesc_none(smem_u32(sBias), 128, 256), idf, 0u);
#pragma unroll
        for (int kk = 0; kk < H / 16; ++kk)
          umma_bf16(t_r, sdesc_sw128(fbase + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                    sdesc_sw128(w0 + (kk >> 2) * (H * 128) + (kk & 3) * 32, 16, 1024), idf, 1u);
        umma_commit(y_full);
      };
      if (count > 0) y_mma(0);
      for (int it = 0; it < count; ++it) {
        const uint32_t fbase = f_base + (it & 1) * TILE;
        const uint32_t acc = it > 0 ? 1u : 0u;
        // e_0(t) = delta_1(t) W_1 / 2 into R (the fused kernel's dX MMA of layer 1)
#ifndef DINR_DW01_NOD1
        mbar_wait(d1_full, it & 1);
#endif
        mbar_wait(y_free, it & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < H / 16; ++kk)
          umma_bf16(t_r, sdesc_sw128(d1 + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), sdesc_sw128(w1 + kk * 2048, H * 128, 1024),
                    idx, kk > 0 ? 1u : 0u);
        umma_commit(e_full);
        // layer 1: dW_1 += delta_1^T h_0, db_1 += delta_1^T 1
        mbar_wait(h_full, it & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t a = (acc || kk > 0) ? 1u : 0u;
          umma_bf16(t_dw1, sdesc_sw128(d1 + kk * 2048, 16384, 1024), sdesc_sw128(hd + kk * 2048, 16384, 1024), idw, a);
          umma_bf16(t_db1, sdesc_sw128(d1 + kk * 2048, 16384, 1024), sdesc_sw128(on + (kk & 3) * 32, 16, 1024), idb, a);
        }
        umma_commit(d1_free);
        umma_commit(h_done);
        if (it + 1 < count) y_mma(it + 1);  // overlaps the delta_0 epilogue
        // layer 0: dW_0 += delta_0^T gamma(x), db_0 += delta_0^T 1
        mbar_wait(d0_full, it & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t a = (acc || kk > 0) ? 1u : 0u;
          umma_bf16(t_dw0, sdesc_sw128(hd + kk * 2048, 16384, 1024), sdesc_sw128(fbase + kk * 2048, 16384, 1024), idw, a);
          umma_bf16(t_db0, sdesc_sw128(hd + kk * 2048, 16384, 1024), sdesc_sw128(on + (kk & 3) * 32, 16, 1024), idb, a);
        }
        umma_commit(&f_free[it & 1]);
        umma_commit(d0_done);
      }
      umma_commit(done);
    }
  } else if (warp >= 2 + LY::NFW) {
    // --------------------------------------------------------------- GRFF feature warps
    const int row = ((warp & 3) << 5) | lane, fh = (warp - 2 - LY::NFW) >> 2;  // frequency half
    const uint32_t f_base = smem_u32(sF);
    constexpr int NFC = (C / 2) / 8;
    int it = 0;
    RayRec rr = grff_fetch(p.rec32, (int64_t)split * 128 + row, p.lg_ns, split < p.n_tiles && (int64_t)split * 128 + row < p.nsamp);
    for (int64_t t = split; t < p.n_tiles; t += ks, ++it) {
      const int64_t g = t * 128 + row;
      const float4 rb = grff_coords_from(rr, g, p.lg_ns, p.n_s, g < p.nsamp, p.jit);
      const int64_t gn = (t + ks) * 128 + row;  // next tile's ray record, in flight meanwhile
      rr = grff_fetch(p.rec32, gn, p.lg_ns, t + ks < p.n_tiles && gn < p.nsamp);
      uint32_t pc[NFC][4], ps[NFC][4];
#pragma unroll
      for (int fc = 0; fc < NFC; ++fc) grff8(sB4, fh * (C / 2) + 8 * fc, rb, pc[fc], ps[fc]);
      const int fb = it & 1;
      if (it >= 2) DW01_WAIT(&f_free[fb], ((it - 2) >> 1) & 1);  // y(t-2), dW_0(t-2) read it
      const uint32_t fbase = f_base + fb * TILE;
#pragma unroll
      for (int fc = 0; fc < NFC; ++fc) {
        const int c0 = fh * (C / 2) + 8 * fc;
        st_shared_v4(fbase + sw128_offset(row, c0, 128), pc[fc][0], pc[fc][1], pc[fc][2], pc[fc][3]);
        st_shared_v4(fbase + sw128_offset(row, C + c0, 128), ps[fc][0], ps[fc][1], ps[fc][2], ps[fc][3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&fbar[fb]);
    }
  } else {
    // --------------------------------------------------------------- Swish / delta_0 warps
    constexpr int NQ = LY::NQ;
    const int row = ((warp & 3) << 5) | lane, half = (warp - 2) >> 2;  // half = column part 0..NQ-1
    const uint32_t hd = smem_u32(sHD);
    const uint32_t trow = t_r + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(half * (H / NQ));
    constexpr int NHC = H / (16 * NQ);
    int it = 0;
    for (int64_t t = split; t < p.n_tiles; t += ks, ++it) {
      // h_0 = swish(y_0), s2_0 = 2 swish'(z_0) of tile t: y = z / 2 from the prescaled MMA,
      // h = y (1 + tanh y), s2 = 1 + t + y (1 - t^2) -- the fused kernel's packed-bf16 arithmetic
      DW01_WAIT(y_full, it & 1);
      tc_fence_after();
      uint32_t hpk[NHC][8], s2k[NHC][8];
#pragma unroll
      for (int hc = 0; hc < NHC; ++hc) {
        uint32_t v[16];
        tmem_ld16(trow + hc * 16, v);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 8; ++i) hpk[hc][i] = pack_bf16x2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(y_free);  // e_0(t) may now be computed into R
#pragma unroll
      for (int hc = 0; hc < NHC; ++hc)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint32_t yb = hpk[hc][i], th = bf2_tanh(yb);
          const uint32_t w = bf2_fma(th, th ^ kBf2Sign, kBf2One);
          s2k[hc][i] = bf2_fma(yb, w, bf2_add(th, kBf2One));
          hpk[hc][i] = bf2_fma(yb, th, yb);
        }
#ifndef DINR_DW01_NOHD
      if (it > 0) DW01_WAIT(d0_done, (it - 1) & 1);
#endif  // dW_0(t-1) has read delta_0(t-1)
#pragma unroll
      for (int hc = 0; hc < NHC; ++hc) {
        const int col0 = half * (H / NQ) + hc * 16;
#pragma unroll
        for (int q = 0; q < 2; ++q)
          st_shared_v4(hd + sw128_offset(row, col0 + 8 * q, 128), hpk[hc][4 * q], hpk[hc][4 * q + 1], hpk[hc][4 * q + 2],
                       hpk[hc][4 * q + 3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(h_full);
      // delta_0 = e_0 s2_0 (e_0 = delta_1 W_1 / 2, s2_0 = 2 swish'(z_0)), rounded as in the fused kernel
      DW01_WAIT(e_full, it & 1);
      tc_fence_after();
#pragma unroll
      for (int hc = 0; hc < NHC; ++hc) {
        uint32_t v[16];
        tmem_ld16(trow + hc * 16, v);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 8; ++i)
#ifdef DINR_F2_PACKED_DELTA
          hpk[hc][i] = bf2_mul(pack_bf16x2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1])), s2k[hc][i]);
#else  // delta_0 = e_0 * swish'(z_0) in fp32, one bf16 rounding (as k_fused2)
          hpk[hc][i] = pack_bf16x2(__uint_as_float(v[2 * i]) * bf16lo(s2k[hc][i]),
                                   __uint_as_float(v[2 * i + 1]) * bf16hi(s2k[hc][i]));
#endif
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(e_free);  // y(t+1) may now be computed into R
#ifndef DINR_DW01_NOHD
      DW01_WAIT(h_done, it & 1);
#endif  // dW_1(t) has read h_0(t)
#pragma unroll
      for (int hc = 0; hc < NHC; ++hc) {
        const int col0 = half * (H / NQ) + hc * 16;
#pragma unroll
        for (int q = 0; q < 2; ++q)
          st_shared_v4(hd + sw128_offset(row, col0 + 8 * q, 128), hpk[hc][4 * q], hpk[hc][4 * q + 1], hpk[hc][4 * q + 2],
                       hpk[hc][4 * q + 3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(d0_full);
    }
  }
  __syncwarp();
  // --------------------------------------------------------------- flush (Swish warps 2-9)
  if (warp >= 2 && warp < 2 + LY::NFW) {
    if (count > 0) {
      DW01_WAIT(done, 0);
      tc_fence_after();
    }
    constexpr int NQ = LY::NQ;
    const int q4 = warp & 3, half = (warp - 2) >> 2, o = (q4 << 5) | lane;
    const uint32_t lanebase = (uint32_t)(q4 * 32) << 16;
    for (int l = 0; l < 2; ++l) {
      float *dst = p.dw_part + (((size_t)l * ks + split) * 128 + o) * H;
#pragma unroll 1
      for (int cb = 0; cb < H / (32 * NQ); ++cb) {
        const int col = half * (H / NQ) + cb * 32;
        uint32_t v[32];
        tmem_ld32((l ? t_dw1 : t_dw0) + lanebase + col, v);
        tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 8; ++q)
          reinterpret_cast<float4 *>(dst + col)[q] =
              count > 0 ? make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                      __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]))
                        : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if (half == 0) {
        uint32_t v[16];
        tmem_ld16((l ? t_db1 : t_db0) + lanebase, v);
        tmem_wait_ld();
        p.db_part[((size_t)l * ks + split) * 128 + o] = count > 0 ? __uint_as_float(v[0]) : 0.f;
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
