// k_tc_dw.cuh -- weight-gradient GEMM on the tensor cores (part of north_star subsystem (3)):
//   dW_l[o][i] = sum_samples delta_l[s][o] h_l[s][i],   db_l[o] = sum_samples delta_l[s][o]
// (eq:partiald via the chain rule).  K = samples is split over CTAs (grid.x);
// grid.y = 128-row output block of o, grid.z = layer.  Operands are the bf16 SW128 tile
// images written by K3 (one 128-sample tile = one K-stage), fetched with 1-D bulk copies
// into a multi-stage mbarrier ring (thread 0 = producer, thread 32 = MMA issuer).
//   A = delta^T : M = o, K = sample, MN-major (LBO = 16 KB between 64-feature blocks)
//   B = h       : N = i, K = sample, MN-major
//   db          : second MMA with B = an all-ones K-major tile (N = 16), column 0 = db.
// fp32 partials are reduced over the K-split in fixed order by k_assemble (deterministic).
#pragma once
#include "internal.cuh"
#include "k_features.cuh"
#include "ptx_sm100.cuh"

namespace dinr {

struct DwParams {
  const uint8_t *hstash, *dstash;
  int64_t n_tiles;
  int L, ksplit, nmb;  // ksplit = partial-slot stride (max of ks0, ks1)
  int ks0, ks1;        // K-splits (CTAs) of layer 0 and of every other layer: grid.x = ks0 + (layers-1) ks1
  float *dw_part, *db_part;
  // feat0: layer 0's input tile (GRFF features) is recomputed from the ray records instead of
  // being read from hstash (fused path: N_s a power of two)
  int feat0;
  const float4 *rec32;
  const float *B;
  int n_s, lg_ns;
  int64_t nsamp;
  Jitter jit;
  // k_tc_dwz (H = 256 split path with k_tc_fwd3): layer inputs h_l (l >= 1) rebuilt from the
  // forward's fp16 y = z / 2 stash
  const uint8_t *ystash;
};

// The tensor core's fp32 accumulation loses precision with the length of the chain of MMAs into
// one TMEM accumulator (measured: the cone512 gradient's deviation from batch linearity grew in
// proportion to the tiles per CTA, 1.3e-3 at 2730 tiles).  Every CTA therefore restarts the
// accumulator every kDwFlushTiles tiles and warps 2-9 add it into fp32 registers (in CTAs whose B
// operand is computed on chip -- layer-0 features, or h from the y stash -- the same warps build it,
// the flushes interleaved with the tiles).
constexpr int kDwFlushTiles = 64;

template <int H>
struct DwLayout {
  static constexpr uint32_t A_STAGE = 32768;  // two 64-feature blocks (second is zero for H = 64)
  static constexpr uint32_t A_COPY = H >= 128 ? 32768u : 16384u;
  static constexpr uint32_t B_STAGE = H * 256;
  static constexpr uint32_t STAGE = A_STAGE + B_STAGE;
  static constexpr int NST = H == 64 ? 4 : (H == 128 ? 3 : 2);
  static constexpr uint32_t TMEM_COLS = H == 64 ? 128 : (H == 128 ? 256 : 512);
  static constexpr int NT = 320;  // warp 0: copies, warp 1: MMA, warps 2-9: features, warps 2-5: epilogue
  static size_t smem_bytes() { return 1024 + (size_t)NST * STAGE + 2048 + (H / 2) * 16 + 256; }
};

template <int H>
__global__ void __launch_bounds__(DwLayout<H>::NT, 1) k_tc_dw(DwParams p) {
  using LY = DwLayout<H>;
  constexpr int NST = LY::NST;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared address space
  uint8_t *ones = smem + NST * LY::STAGE;
  float4 *sB4 = reinterpret_cast<float4 *>(ones + 2048);
  uint64_t *full = reinterpret_cast<uint64_t *>(sB4 + H / 2);
  uint64_t *empty = full + NST;
  uint64_t *done = empty + NST;
  uint64_t *flush_full = done + 1, *flush_free = done + 2;  // accumulator chunk complete / read out
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(done + 3);

  const int tid = threadIdx.x, warp = tid >> 5;
  const int bx = blockIdx.x, mb = blockIdx.y;
  const int l = bx < p.ks0 ? 0 : 1 + (bx - p.ks0) / p.ks1;
  const int split = bx < p.ks0 ? bx : (bx - p.ks0) % p.ks1;
  const int ks = l == 0 ? p.ks0 : p.ks1;
  const bool feat = p.feat0 && l == 0;
  const bool fl = true;  // chunked accumulation (warps 2-9 flush every kDwFlushTiles tiles)
  if (warp == 0) {
    tmem_alloc(tmem_slot, LY::TMEM_COLS);
    tmem_relinquish();
  }
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], feat ? 1 + 8 : 1);  // + one arrival per feature warp
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    mbar_init(flush_full, 1);
    mbar_init(flush_free, 8);
    fence_mbar_init();
  }
  // constant operands: all-ones tile (bf16 1.0 = 0x3F80) and, for H = 64, zero pad blocks
  for (int i = tid; i < 2048 / 4; i += LY::NT) reinterpret_cast<uint32_t *>(ones)[i] = 0x3F803F80u;
  if (feat)
    for (int i = tid; i < H / 2; i += LY::NT) sB4[i] = reinterpret_cast<const float4 *>(p.B)[i];
  if (H == 64)
    for (int s = 0; s < NST; ++s)
      for (int i = tid; i < 16384 / 16; i += LY::NT)
        reinterpret_cast<uint4 *>(smem + s * LY::STAGE + 16384)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tmem_dw = tmem, tmem_db = tmem + H;

  int count = 0;
  for (int64_t t = split; t < p.n_tiles; t += ks) ++count;

  if (tid == 0) {
    int it = 0;
    for (int64_t t = split; t < p.n_tiles; t += ks, ++it) {
      int st = it % NST;
      if (it >= NST) mbar_wait(&empty[st], ((it / NST) - 1) & 1);
      uint8_t *sa = smem + st * LY::STAGE, *sb = sa + LY::A_STAGE;
      mbar_arrive_expect_tx(&full[st], LY::A_COPY + (feat ? 0u : LY::B_STAGE));
      const uint8_t *dsrc = p.dstash + ((size_t)l * p.n_tiles + t) * (H * 256) + (size_t)mb * 32768;
      const uint8_t *hsrc = p.hstash + ((size_t)l * p.n_tiles + t) * (H * 256);
      bulk_g2s(sa, dsrc, LY::A_COPY, &full[st]);
      if (!feat)
        for (uint32_t off = 0; off < LY::B_STAGE; off += 32768u)
          bulk_g2s(sb + off, hsrc + off, min(32768u, LY::B_STAGE - off), &full[st]);
    }
  } else if (tid == 32) {
    const uint32_t id_dw = idesc_bf16(128, H, 1, 1);
    const uint32_t id_db = idesc_bf16(128, 16, 1, 0);
    const uint32_t ones_a = smem_u32(ones);
    for (int it = 0; it < count; ++it) {
      int st = it % NST;
      const int ci = fl ? it % kDwFlushTiles : it;  // tile index within the accumulator chunk
      mbar_wait(&full[st], (it / NST) & 1);
      if (fl && ci == 0 && it > 0) mbar_wait(flush_free, ((it / kDwFlushTiles) - 1) & 1);
      tc_fence_after();
      uint32_t sa = smem_u32(smem + st * LY::STAGE), sb = sa + LY::A_STAGE;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        uint64_t ad = sdesc_sw128(sa + kk * 2048, 16384, 1024);
        uint64_t bd = sdesc_sw128(sb + kk * 2048, 16384, 1024);
        uint64_t od = sdesc_sw128(ones_a + (kk & 3) * 32, 16, 1024);
        uint32_t acc = (ci > 0 || kk > 0) ? 1u : 0u;
        umma_bf16(tmem_dw, ad, bd, id_dw, acc);
        umma_bf16(tmem_db, ad, od, id_db, acc);
      }
      umma_commit(&empty[st]);
      if (fl && (ci == kDwFlushTiles - 1 || it == count - 1)) umma_commit(flush_full);
    }
    umma_commit(done);
  }
  if (fl && warp >= 2 && warp < 10) {
    // flush warps: thread = (accumulator lane o, column half cp); every chunk of kDwFlushTiles
    // tiles is added into fp32 registers, then the partial row is written from them
    const int q4 = warp & 3, cp = (warp - 2) >> 2, o = (q4 << 5) | (tid & 31);
    const uint32_t trow = (uint32_t)(q4 * 32) << 16;
    float racc[H / 2], rdb = 0.f;
#pragma unroll
    for (int i = 0; i < H / 2; ++i) racc[i] = 0.f;
    const int nch = (count + kDwFlushTiles - 1) / kDwFlushTiles;
    int c0 = 0;
    if (feat) {
      // layer 0's B operand built on chip, interleaved with the accumulator flushes: chunk c is
      // flushed before the tile that would need the stage its restart holds back
      int it = 0;
      for (int64_t t = split; t < p.n_tiles; t += ks, ++it) {
        while (c0 < nch && c0 * kDwFlushTiles + kDwFlushTiles - 1 <= it - NST) {
          mbar_wait(flush_full, c0 & 1);
          tc_fence_after();
#pragma unroll
          for (int cb = 0; cb < H / 64; ++cb) {
            uint32_t v[32];
            tmem_ld32(tmem_dw + trow + cp * (H / 2) + cb * 32, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) racc[cb * 32 + i] += __uint_as_float(v[i]);
          }
          if (cp == 0) {
            uint32_t v[16];
            tmem_ld16(tmem_db + trow, v);
            tmem_wait_ld();
            rdb += __uint_as_float(v[0]);
          }
          tc_fence_before();
          __syncwarp();
          if ((tid & 31) == 0) mbar_arrive(flush_free);
          ++c0;
        }
        const int st = it % NST;
        const uint32_t sb = smem_u32(smem + st * LY::STAGE + LY::A_STAGE);
        // layer 0: B = gamma(x) of the tile's 128 samples, the same SW128 image the forward fed to
        // its layer-0 MMA (thread = sample row o, frequency half cp)
        constexpr int C = H / 2;
        const int64_t g = t * 128 + o;
        const float4 rb = grff_coords(p.rec32, g, p.lg_ns, p.n_s, g < p.nsamp, p.jit);
        if (it >= NST) mbar_wait(&empty[st], ((it / NST) - 1) & 1);
#pragma unroll
        for (int f0 = cp * (C / 2); f0 < (cp + 1) * (C / 2); f0 += 8) {
          uint32_t pc[4], ps[4];
          grff8(sB4, f0, rb, pc, ps);
          st_shared_v4(sb + sw128_offset(o, f0, 128), pc[0], pc[1], pc[2], pc[3]);
          st_shared_v4(sb + sw128_offset(o, C + f0, 128), ps[0], ps[1], ps[2], ps[3]);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(&full[st]);
      }
    }
    for (int c = c0; c < nch; ++c) {
      mbar_wait(flush_full, c & 1);
      tc_fence_after();
#pragma unroll
      for (int cb = 0; cb < H / 64; ++cb) {
        uint32_t v[32];
        tmem_ld32(tmem_dw + trow + cp * (H / 2) + cb * 32, v);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) racc[cb * 32 + i] += __uint_as_float(v[i]);
      }
      if (cp == 0) {
        uint32_t v[16];
        tmem_ld16(tmem_db + trow, v);
        tmem_wait_ld();
        rdb += __uint_as_float(v[0]);
      }
      tc_fence_before();
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(flush_free);
    }
    const bool live = (H >= 128) || o < 64;
    if (live) {
      float *dst = p.dw_part + ((((size_t)l * p.nmb + mb) * p.ksplit + split) * 128 + o) * H + cp * (H / 2);
#pragma unroll
      for (int q = 0; q < H / 8; ++q)
        reinterpret_cast<float4 *>(dst)[q] = make_float4(racc[4 * q], racc[4 * q + 1], racc[4 * q + 2], racc[4 * q + 3]);
      if (cp == 0) p.db_part[(((size_t)l * p.nmb + mb) * p.ksplit + split) * 128 + o] = rdb;
      // slots this layer does not use (ks < ksplit) are zero for the fixed-order reduction
      for (int s2 = split + ks; s2 < p.ksplit; s2 += ks) {
        float4 *z = reinterpret_cast<float4 *>(p.dw_part + ((((size_t)l * p.nmb + mb) * p.ksplit + s2) * 128 + o) * H + cp * (H / 2));
        for (int q = 0; q < H / 8; ++q) z[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (cp == 0) p.db_part[(((size_t)l * p.nmb + mb) * p.ksplit + s2) * 128 + o] = 0.f;
      }
    }
  }
  __syncwarp();
  if (count > 0) {
    mbar_wait(done, 0);
    tc_fence_after();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, LY::TMEM_COLS);
  }
}

}  // namespace dinr
