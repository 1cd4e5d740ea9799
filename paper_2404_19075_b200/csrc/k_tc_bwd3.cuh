// k_tc_bwd3.cuh -- split-path backward dX chain (K3) for H = 256 on CTA pairs (cta_group::2),
// north_star subsystem (3) (eq:partiald): the backward twin of k_tc_fwd3.
//
// Pair-iteration pi = 512 samples = 4 tiles, stream s / CTA rank r owns tile 4 pi + 2 s + r.
// Per layer l = L-1 .. 1 the leader issues, for (s, h) = (0,0) (0,1) (1,0) (1,1), 16 pair MMAs
// M = 256 (samples), N = 128 (input features [128 h, 128 h + 128) of layer l; the leader holds
// the 64-column block 2h of the MN-major W_l image, the peer block 2h + 1), K = 256 (the layer's
// output features):  e_{l-1} = delta_l W_l.  Same math, rounding and outputs as k_tc_mlp MODE 2:
// the top layer's delta and head gradients from the stashed fp16 z_{L-1} and the upstream u,
// then delta_{l-1} = e_{l-1} (.) swish'(z_{l-1}) (bf16 swish' from the forward's stash), every
// delta_l image bulk-stored to the delta stash for the dW GEMM (k_tc_dw.cuh).
//   warps 0-7: stream 0 epilogue, warps 8-15: stream 1 (thread = sample row x column half)
//   warp 16 lane 0: MMA issue (leader)     warp 17 lane 0: W loads     warp 18 lane 0: delta stores
//   warp 19 lane 0: (peer) passes its landed W K-halves on to the leader's w_full
// Barriers as in k_tc_fwd3; acc_full[s] = the stream's dX MMAs retired + this CTA's delta store
// read A_s (the store thread arrives twice after delta_0, which no MMA follows).
#pragma once
#include "internal.cuh"
#include "k_tc_mlp.cuh"
#include "ptx_sm100.cuh"

namespace dinr {

// stash copies stream through L2 (evict_first): they are read back by a later kernel, 21 GB later
#ifndef STASH_S2G
#define STASH_S2G(d, s_, n) bulk_s2g_hint(d, s_, n, policy_evict_first())
#endif

// The W blocks move through a ring of B3_WRING K-half buffers (rows [128 kh, +128) of this CTA's
// 64-column block of piece h, 16 KB): K-half j of the kernel's sequence (layer, piece, K-half; both
// streams use it) in buffer j mod B3_WRING, so the next layer's first K-half loads while the
// current layer runs (as k_tc_fwd3).
#ifndef B3_WRING
#define B3_WRING 5
#endif
// 1: the delta store of a stream-layer starts with K-blocks 0 and 2 (the first half of every epilogue
// thread's columns) as soon as the epilogue has written them, so the copy that the next layer's
// epilogue waits for is half as long; 0: one 64 KB copy after the whole epilogue
#ifndef B3_SPLIT
#define B3_SPLIT 1
#endif
// 1 (with B3_SPLIT): the two column halves of a stream interleave their 16-column chunks (thread
// column half cg takes chunks 2k + cg), so the K-blocks of A_s complete one after another and each
// is copied as soon as it is written: the copy the next layer waits for is one 16 KB K-block
#ifndef B3_QSPLIT
#define B3_QSPLIT 1
#endif
struct Bwd3Layout {
  static constexpr int H = 256;
  static constexpr int NT = 512 + 128;
  static constexpr int NWB = B3_WRING;
  static constexpr uint32_t A_BYTES = H * 256u;   // 128 rows x 256 bf16
  static constexpr uint32_t WQ_BYTES = H * 128u;  // one 64-column block of W_l: 256 rows x 128 B
  static constexpr uint32_t WH_BYTES = WQ_BYTES / 2;  // one K-half of it
  static size_t smem_bytes() {
    return 1024 + 2 * (size_t)A_BYTES + NWB * (size_t)WH_BYTES + (H + 4) * 4 + 2 * 8 * (H + 1) * 4 + 256;
  }
};

__global__ void __launch_bounds__(Bwd3Layout::NT, 1) k_tc_bwd3(TcParams p, int nhead_slots) {
  using LY = Bwd3Layout;
  constexpr int H = LY::H;
  constexpr uint32_t A_BYTES = LY::A_BYTES, W_LAYER = H * H * 2u, WQ = LY::WQ_BYTES, WH = LY::WH_BYTES;
  constexpr int NWB = LY::NWB;
  constexpr int NCB = H / 64;                 // 32-column chunks of a thread's column half
  constexpr uint32_t kZTile = 128u * H * 2u;  // one tile of the 16-bit backward state
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // same offsets in both CTAs
  const int L = p.L;
  uint8_t *sA0 = smem;                              // A tiles (delta_l images) of streams 0, 1
  uint8_t *sW = sA0 + 2 * A_BYTES;                  // NWB W K-half buffers: [128 output rows][128 B]
  float *sWo = reinterpret_cast<float *>(sW + NWB * WH);  // w_o[H], b_o
  float *red = sWo + H + 4;                          // [16 warps][H + 1] head partials
  uint64_t *bars = reinterpret_cast<uint64_t *>(red + 2 * 8 * (H + 1));
  uint64_t *w_full = bars, *w_loc = bars + NWB, *w_free = bars + 2 * NWB;  // [NWB] each
  uint64_t *a_full = bars + 3 * NWB, *a_rdy = a_full + 2, *acc_full = a_full + 4;  // [2] each
  // h_rdy[s][kb]: K-block kb of A_s written (kb 0..2; with halves only [s][0]: K-blocks 0 and 2).
  // One barrier per K-block, so none can run more than one phase ahead of the store thread, which
  // serves the streams in turn.
  uint64_t *h_rdy = a_full + 6;                                                    // [2][3]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(a_full + 12);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  if (tid == 512) {
    for (int i = 0; i < NWB; ++i) {
      mbar_init(&w_full[i], 2);
      mbar_init(&w_loc[i], 1);
      mbar_init(&w_free[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&a_full[i], 2);
      mbar_init(&a_rdy[i], 1);
      mbar_init(&acc_full[i], 2);
      for (int kb = 0; kb < 3; ++kb) mbar_init(&h_rdy[i * 3 + kb], 8);  // one arrival per epilogue warp of the stream
    }
    fence_mbar_init();
  }
  const int64_t per = (int64_t)H * H + H;
  for (int i = tid; i <= H; i += LY::NT) sWo[i] = p.params[(int64_t)L * per + i];
  cluster_sync();
  if (warp == 0) {
    tmem_alloc_pair(tmem_slot, 512);
    tmem_relinquish_pair();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t n_iter = p.n_tiles / 4;
  const int64_t cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  float head_acc[2 * NCB];  // per 16-column chunk of the thread's half: lanes l, l ^ 16 hold column l & 15
#pragma unroll
  for (int i = 0; i < 2 * NCB; ++i) head_acc[i] = 0.f;
  float bo_acc = 0.f;

  if (tid == 512) {
    if (leader && L >= 2) {
      // ============================================================ MMA issue (leader)
      const uint32_t a_base0 = smem_u32(sA0), w_base = smem_u32(sW);
      const uint32_t idesc = idesc_bf16(256, 128, 0, 1);  // A K-major (delta rows), B MN-major (W_l)
      uint32_t aph[2] = {0, 0};
      uint32_t lay = 0;  // dX layers processed so far (W buffer phase)
      for (int64_t pi = cl; pi < n_iter; pi += ncl) {
        for (int l = L - 1; l >= 1; --l, ++lay) {
          for (int s = 0; s < 2; ++s) {
            for (int h = 0; h < 2; ++h) {
              // K-halves of this CTA's block of W_l piece h (for both streams): waited for by stream
              // 0's step, released after stream 1's
              if (h == 0) {
                mbar_wait_cluster(&a_full[s], aph[s]);
                aph[s] ^= 1;
              }
              const uint32_t a_base = a_base0 + s * A_BYTES;
              for (int kh = 0; kh < 2; ++kh) {
                const uint32_t j = (lay * 2 + h) * 2 + kh, b = j % NWB;
                if (s == 0) mbar_wait_cluster(&w_full[b], (j / NWB) & 1);
                tc_fence_after();
                const uint32_t wb = w_base + b * WH;
#pragma unroll 4
                for (int kk = 8 * kh; kk < 8 * kh + 8; ++kk) {  // K = the layer's output features (16 rows of W_l)
                  uint64_t ad = sdesc_sw128(a_base + (kk >> 2) * (128 * 128) + (kk & 3) * 32, 16, 1024);
                  uint64_t bd = sdesc_sw128(wb + (kk - 8 * kh) * 2048, WH, 1024);
                  umma_bf16_pair(tmem + s * 256 + h * 128, ad, bd, idesc, kk > 0 ? 1u : 0u);
                }
                if (s == 1) umma_commit_pair(&w_free[b], 3);
              }
              if (h == 1) umma_commit_pair(&acc_full[s], 3);
            }
          }
        }
      }
    }
  } else if (tid == 544) {
    // ============================================================ W loads (both CTAs)
    const uint8_t *wsrc = reinterpret_cast<const uint8_t *>(p.wpack);
    uint32_t lay = 0;
    for (int64_t pi = cl; pi < n_iter; pi += ncl) {
      for (int l = L - 1; l >= 1; --l, ++lay) {
        for (int h = 0; h < 2; ++h) {
          for (int kh = 0; kh < 2; ++kh) {
            const uint32_t j = (lay * 2 + h) * 2 + kh, b = j % NWB;
            if (j >= NWB) mbar_wait_long(&w_free[b], ((j / NWB) - 1) & 1);  // stream 1's MMAs on K-half j - NWB
            uint64_t *bar = leader ? &w_full[b] : &w_loc[b];
            mbar_arrive_expect_tx(bar, WH);
            // rows [128 kh, +128) of this CTA's 64-column block 2h + r of the MN-major W_l image
            bulk_g2s(sW + b * WH, wsrc + (size_t)l * W_LAYER + (size_t)(2 * h + rank) * WQ + kh * WH, WH, bar);
          }
        }
      }
    }
  } else if (tid == 608) {
    // ============================================================ peer: W halves landed -> leader
    if (!leader) {
      const uint32_t w_full_leader = mapa_shared(smem_u32(&w_full[0]), 0);
      uint32_t lay = 0;
      for (int64_t pi = cl; pi < n_iter; pi += ncl)
        for (int l = L - 1; l >= 1; --l, ++lay)
          for (uint32_t j = lay * 4; j < lay * 4 + 4; ++j) {
            const uint32_t b = j % NWB;
            mbar_wait_long(&w_loc[b], (j / NWB) & 1);
            mbar_arrive_remote(w_full_leader + b * 8);
          }
    }
  } else if (tid == 576) {
    // ============================================================ delta-stash stores (both CTAs)
    uint32_t rph[2] = {0, 0}, hph[2] = {0, 0};  // (every h_rdy[s][kb] completes once per store: one parity per stream)
    constexpr uint32_t KB = A_BYTES / 4;  // one 64-column K-block of the image
    for (int64_t pi = cl; pi < n_iter; pi += ncl) {
      for (int l = L - 1; l >= 0; --l) {
        for (int s = 0; s < 2; ++s) {
          const int64_t tile = 4 * pi + 2 * s + rank;
          uint8_t *dst = p.dstash + ((size_t)l * p.n_tiles + tile) * A_BYTES;
          const uint8_t *src = sA0 + s * A_BYTES;
#if B3_SPLIT && B3_QSPLIT
          for (int kb = 0; kb < 3; ++kb) {  // K-blocks 0, 1, 2 as the epilogue completes them
            mbar_wait_long(&h_rdy[s * 3 + kb], hph[s]);
#ifndef DINR_DBG_K3_NOSTORE
            STASH_S2G(dst + kb * KB, src + kb * KB, KB);
            bulk_commit();
#endif
          }
          hph[s] ^= 1;
#elif B3_SPLIT
          mbar_wait_long(&h_rdy[s * 3], hph[s]);
          hph[s] ^= 1;
#ifndef DINR_DBG_K3_NOSTORE
          STASH_S2G(dst, src, KB);
          STASH_S2G(dst + 2 * KB, src + 2 * KB, KB);
          bulk_commit();
#endif
#endif
          mbar_wait_long(&a_rdy[s], rph[s]);
          rph[s] ^= 1;
#ifndef DINR_DBG_K3_NOSTORE  // timing experiment only (the dW GEMM then reads a stale delta stash)
#if B3_SPLIT && B3_QSPLIT
          STASH_S2G(dst + 3 * KB, src + 3 * KB, KB);
#elif B3_SPLIT
          STASH_S2G(dst + KB, src + KB, KB);
          STASH_S2G(dst + 3 * KB, src + 3 * KB, KB);
#else
          STASH_S2G(dst, src, A_BYTES);
#endif
          bulk_commit();
          bulk_wait_read_all();
#endif
          mbar_arrive(&acc_full[s]);
          if (l == 0) mbar_arrive(&acc_full[s]);  // no MMA follows delta_0
        }
      }
    }
    bulk_wait_all();
  } else if (tid < 512) {
    // ============================================================ epilogue streams
    const int s = tid >> 8, wt = tid & 255;
    const int row = wt & 127, cg = wt >> 7;
    const int cb_lo = cg * NCB;
    // the thread's k-th 16-column chunk
    auto c16_of = [&](int k) { return B3_SPLIT && B3_QSPLIT ? 2 * k + cg : cb_lo * 2 + k; };
    // K-block written: 0 and 2 at k = NCB - 1 (halves), or K-block (k - 1) / 2 at odd k (interleaved)
    auto kblock_done = [&](int k) { return B3_SPLIT && (B3_QSPLIT ? ((k & 1) && k < 2 * NCB - 1) : k == NCB - 1); };
    const uint32_t a_base = smem_u32(sA0) + s * A_BYTES;
    const uint32_t tmem_row = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(s * 256);
    const uint32_t a_full_leader = mapa_shared(smem_u32(&a_full[s]), 0);
    const uint64_t pol_z = policy_evict_first();
    uint32_t accph = 0;
    bool a_busy = false;  // A_s still read by the previous iteration's delta_0 store
    // A_s written -> this CTA's delta store and (unless it is delta_0, which no MMA reads) the
    // pair MMA.  delta_0 must not arrive on a_full: the MMA thread never waits for it, and the next
    // iteration's top-layer hand-off could otherwise complete a second phase before it looks.
    // K-blocks 0 and 2 of A_s written (every thread's first four 16-column chunks) -> the delta
    // store may start on them
    [[maybe_unused]] auto half_off = [&](int kb) {
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&h_rdy[s * 3 + kb]);
    };
    auto hand_off = [&](bool to_mma) {
      fence_proxy_async_smem();
      asm volatile("bar.sync %0, 256;" ::"r"(1 + s) : "memory");
      if (wt == 0) {
        mbar_arrive(&a_rdy[s]);
        if (!to_mma) {
        } else if (leader)
          mbar_arrive(&a_full[s]);
        else
          mbar_arrive_remote(a_full_leader);
      }
    };
    for (int64_t pi = cl; pi < n_iter; pi += ncl) {
      const int64_t tile = 4 * pi + 2 * s + rank;
      const int64_t g = tile * 128 + row;
      const bool valid = g < p.nsamp;
      // ---------------------------------------------------------------- top layer (as K3)
      const float u_row = valid ? p.u[ray_of(g, p.n_s)] : 0.f;
      {
        const uint8_t *zsrc = p.zstash + (((size_t)(L - 1) * p.n_tiles + tile) * (H / 16) * 128 + row) * 32;
        uint4 zt[2][2];
        ld_global_v8_hint(zsrc + (size_t)c16_of(0) * 128 * 32, zt[0][0], zt[0][1], pol_z);
        if (a_busy) {
          mbar_wait_long(&acc_full[s], accph);  // CTA scope: TMEM + own smem only
          accph ^= 1;
        }
        a_busy = true;
#pragma unroll
        for (int k = 0; k < 2 * NCB; ++k) {
          const int c16 = c16_of(k);
          if (k + 1 < 2 * NCB)
            ld_global_v8_hint(zsrc + (size_t)c16_of(k + 1) * 128 * 32, zt[(k + 1) & 1][0], zt[(k + 1) & 1][1], pol_z);
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
          if (kblock_done(k)) half_off(B3_QSPLIT ? (k >> 1) : 0);
        }
        if (cg == 0) {
          float us = u_row;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) us += __shfl_xor_sync(0xffffffffu, us, o);
          bo_acc += us;
        }
        hand_off(L >= 2);
      }
      // ---------------------------------------------------------------- dX chain
      for (int l = L - 1; l >= 1; --l) {
        const uint8_t *zsrc = p.zstash + (((size_t)(l - 1) * p.n_tiles + tile) * (H / 16) * 128 + row) * 32;
        uint4 zq[2 * NCB][2];
#ifdef DINR_DBG_K3_NOLOAD  // timing experiment only (swish' = 1)
#pragma unroll
        for (int k = 0; k < 2 * NCB; ++k) zq[k][0] = zq[k][1] = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
#define ld_global_v8_hint(...) (void)0
#endif
#pragma unroll
        for (int k = 0; k < NCB; ++k) ld_global_v8_hint(zsrc + (size_t)c16_of(k) * 128 * 32, zq[k][0], zq[k][1], pol_z);
        if (l >= 2 && cg == 0 && (row & 31) == 0)  // the next step's state into L2 meanwhile
          bulk_prefetch_l2(p.zstash + ((size_t)(l - 2) * p.n_tiles + tile) * kZTile + (size_t)(row >> 5) * (kZTile / 4),
                           kZTile / 4);
        mbar_wait_long(&acc_full[s], accph);  // CTA scope: TMEM + own smem only
        accph ^= 1;
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < 2 * NCB; ++k) {
          const int c16 = c16_of(k);
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
          if (kblock_done(k)) half_off(B3_QSPLIT ? (k >> 1) : 0);
          if (k + NCB < 2 * NCB)  // NCB chunks ahead, into the registers chunk k just released
            ld_global_v8_hint(zsrc + (size_t)c16_of(k + NCB) * 128 * 32, zq[k + NCB][0], zq[k + NCB][1], pol_z);
        }
        tc_fence_before();
        hand_off(l >= 2);
      }
    }
    if (a_busy) {  // the last delta_0 store has read A_s
      mbar_wait_long(&acc_full[s], accph);  // CTA scope: TMEM + own smem only
      accph ^= 1;
    }
  }
  // ------------------------------------------------------------ per-CTA head partials
  __syncthreads();
  if (tid < 512) {
    const int s = tid >> 8, wt = tid & 255, cg = wt >> 7, w8 = wt >> 5;
    if (lane < 16)
#pragma unroll
      for (int k = 0; k < 2 * NCB; ++k)
        red[(s * 8 + w8) * (H + 1) + (B3_SPLIT && B3_QSPLIT ? 2 * k + cg : cg * NCB * 2 + k) * 16 + lane] = head_acc[k];
    if (lane == 0) red[(s * 8 + w8) * (H + 1) + H] = bo_acc;  // (zero for column-half-1 warps)
  }
  __syncthreads();
  for (int k = tid; k <= H; k += LY::NT) {
    float acc = 0.f;
    // the warps of the column half that holds column k (chunks 2k' + cg when interleaved)
    const int w0 = (k < H && (B3_SPLIT && B3_QSPLIT ? ((k >> 4) & 1) : k >= H / 2)) ? 4 : 0;
    for (int s = 0; s < 2; ++s)
      for (int w = w0; w < w0 + 4; ++w) acc += red[(s * 8 + w) * (H + 1) + k];
    p.head_part[(size_t)blockIdx.x * (H + 1) + k] = acc;
    for (int b = blockIdx.x + gridDim.x; b < nhead_slots; b += gridDim.x) p.head_part[(size_t)b * (H + 1) + k] = 0.f;
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 512);
  }
}

}  // namespace dinr
