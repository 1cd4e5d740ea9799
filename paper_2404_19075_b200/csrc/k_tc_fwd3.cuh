// k_tc_fwd3.cuh -- split-path training forward (K2) for H = 256 on CTA pairs (cta_group::2),
// north_star subsystem (2) (a5-a9 for the training step; eq:estforwmod).
//
// Why pairs.  k_tc_fwd2 (one SM, two 128-sample tile streams) spends about half of its epilogue
// time waiting for MMAs that wait for weights: the two 64 KB A tiles leave room for one 64 KB
// W_l N-half, so every half is loaded while the tensor core idles, and the two streams share each
// half, so both epilogues run at the same time instead of during the other stream's MMAs.  On a
// CTA pair a tcgen05.mma.cta_group::2 with M = 256 takes A rows [0, 128) from the leader's shared
// memory and [128, 256) from the peer's, and B columns [0, N/2) / [N/2, N) likewise: each SM holds
// half of every W_l N-half (32 KB), so a ring of weight buffers fits beside the A tiles and the
// next weight load runs under the current MMA, and the two tile streams can run one after the other
// (stream 0's epilogue under stream 1's MMAs and vice versa).
//
// Work unit: pair-iteration pi = 512 samples = 4 tiles; stream s, CTA rank r owns tile 4 pi + 2 s + r
// (TMEM lanes = its 128 samples).  Per layer l the leader issues, for (s, h) = (0,0) (0,1) (1,0)
// (1,1): 16 MMAs M = 256, N = 128 (output features [128 h, 128 h + 128)), K = 256, into TMEM
// columns [256 s + 128 h, +128) of both CTAs.  Each piece is loaded once per layer for both
// streams, as two K-halves through the ring of F3_WRING buffers (below), so the next layer's
// weights load while stream 1 finishes and stream 0's epilogue runs.  Same math, rounding and outputs as k_tc_fwd2 /
// k_tc_mlp MODE 1 (ray-chunk sums of M, h_l images to the h stash, swish'(z_l) / z_{L-1} to the
// s2 stash).
//   warps 0-7: stream 0 epilogue, warps 8-15: stream 1 (thread = sample row x column half)
//   warp 16 lane 0: MMA issue (leader CTA only)
//   warp 17 lane 0: W loads of this CTA's half (both CTAs)
//   warp 18 lane 0: h-stash bulk stores of this CTA's tiles (both CTAs)
//   warp 19 lane 0: (peer) passes its landed W K-halves on to the leader's w_full
// Barriers (per CTA unless noted):
//   w_full[b]   leader only: its own half loaded (expect_tx) + the peer's half loaded (remote arrive)
//   w_loc[b]    peer only: its own half loaded
//   w_free[b]   stream 1's MMAs on ring buffer b retired (multicast commit to both CTAs)
//   a_full[s]   leader only: A_s written by both CTAs' stream-s epilogues (1 local + 1 remote arrive)
//   a_rdy[s]    A_s written by this CTA's epilogue (for its stash store thread)
//   acc_full[s] stream s's layer retired (multicast commit) and this CTA's stash store read A_s
#pragma once
#include "internal.cuh"
#include "k_features.cuh"
#include "k_tc_mlp.cuh"
#include "ptx_sm100.cuh"

namespace dinr {

// stash copies stream through L2 (evict_first): they are read back by a later kernel, 21 GB later
#ifndef STASH_S2G
#define STASH_S2G(d, s_, n) bulk_s2g_hint(d, s_, n, policy_evict_first())
#endif

#ifdef DINR_PHASES
#define F3_T0() const long long _t0 = clock64()
#define F3_ACC(v) (v) += (unsigned long long)(clock64() - _t0)
#else
#define F3_T0() (void)0
#define F3_ACC(v) (void)0
#endif

// Each stream-layer's N = 256 output features run as NP pieces of N = 256 / NP (one pair MMA chain per
// piece); each CTA holds 128 / NP rows of a piece's W block (this CTA's half), in NWB ring buffers
// (64 KB in total), so loads run NWB - 1 pieces ahead of the MMAs.  NP = 2 (N = 128, two 32 KB
// buffers) is the default: NP = 4 (N = 64, four 16 KB buffers, a deeper weight pipeline) measured
// slower (cone4d2048 forward 5.5 -> 7.4 ms): an M = 256, N = 64 pair MMA reads 5 KB of operands per
// 32 cycles from each SM's shared memory, above its 128 B/clk.
#ifndef F3_PIECES
#define F3_PIECES 2
#endif
// The W pieces move through a ring of F3_WRING K-half buffers (this CTA's rows of a piece for 128 of
// the 256 K, 16 KB): K-half j of the kernel's sequence (layer-major, piece, K-half; both streams use
// it) in buffer j mod F3_WRING.  Five buffers (80 KB) let the next layer's first K-half load while
// the current layer runs; two whole-piece buffers (64 KB) made the MMA wait ~2.4 K cycles per layer
// for weights that could only start loading after stream 1's MMAs on the previous layer retired.
#ifndef F3_WRING
#define F3_WRING 5
#endif
struct Fwd3Layout {
  static constexpr int H = 256, C = 128;
  static constexpr int NP = F3_PIECES;             // N pieces per stream-layer
  static constexpr int NWB = F3_WRING;             // K-half W buffers, shared by both streams
  static constexpr int PN = H / NP;                // N of one piece (pair MMA)
  static constexpr int PR = PN / 2;                // W rows per CTA per piece
  static constexpr int NT = 512 + 128;
  static constexpr uint32_t A_BYTES = H * 256u;    // 128 rows x 256 bf16
  static constexpr uint32_t WQ_BYTES = PR * 256u;  // this CTA's rows of a piece for one K-half: PR rows x 128 K
  static size_t smem_bytes(int L) {
    return 1024 + 2 * (size_t)A_BYTES + NWB * (size_t)WQ_BYTES + (size_t)L * H * 4 + (H + 4) * 4 + C * 16 +
           2 * 2 * 128 * 4 + 512;
  }
};

__global__ void __launch_bounds__(Fwd3Layout::NT, 1) k_tc_fwd3(TcParams p) {
  using LY = Fwd3Layout;
  constexpr int H = LY::H, C = LY::C;
  constexpr uint32_t A_BYTES = LY::A_BYTES, W_LAYER = H * H * 2u, WQ = LY::WQ_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // same offsets in both CTAs
  const int L = p.L;
  uint8_t *sA0 = smem;                            // A tiles of streams 0, 1
  uint8_t *sW = sA0 + 2 * A_BYTES;                // NWB W buffers: [4 K-blocks][PR rows][128 B]
  float *sBias = reinterpret_cast<float *>(sW + LY::NWB * WQ);
  float *sWo = sBias + L * H;                     // w_o[H], b_o
  float *sB = sWo + H + 4;                        // C x 4
  float *sMu = sB + C * 4;                        // [2 streams][2 column halves][128 rows]
  uint64_t *bars = reinterpret_cast<uint64_t *>(sMu + 2 * 2 * 128);
  constexpr int NWB = LY::NWB, NP = LY::NP, PN = LY::PN, PR = LY::PR;
  uint64_t *w_full = bars, *w_loc = bars + NWB, *w_free = bars + 2 * NWB;  // [NWB] each
  uint64_t *a_full = bars + 3 * NWB, *a_rdy = a_full + 2, *acc_full = a_full + 4;  // [2] each
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(a_full + 6);

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
    }
    fence_mbar_init();
  }
  const int64_t per = (int64_t)H * H + H;
  // the epilogue works on y = z / 2 = 0.5 acc + 0.5 b (one FFMA), so the bias is stored halved
  const float bscale = 0.5f;
  for (int i = tid; i < L * H; i += LY::NT) sBias[i] = bscale * p.params[(i / H) * per + (int64_t)H * H + (i % H)];
  for (int i = tid; i <= H; i += LY::NT) sWo[i] = p.params[(int64_t)L * per + i];
  for (int i = tid; i < C * 4; i += LY::NT) sB[i] = p.B[i];
  cluster_sync();  // barriers of both CTAs initialized before any remote arrive
  if (warp == 0) {
    tmem_alloc_pair(tmem_slot, 512);
    tmem_relinquish_pair();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t n_iter = p.n_tiles / 4;  // the plan rounds the tile count up to a multiple of 4
  const int64_t cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  if (tid == 512) {
    if (leader) {
      // ============================================================ MMA issue (leader)
      const uint32_t a_base0 = smem_u32(sA0), w_base = smem_u32(sW);
      const uint32_t idesc = idesc_bf16(256, PN, 0, 0);
      uint32_t aph[2] = {0, 0};
      uint32_t lay = 0;  // layers processed so far (W buffer phase)
      [[maybe_unused]] unsigned long long ph_w = 0, ph_a = 0;
      for (int64_t pi = cl; pi < n_iter; pi += ncl) {
        for (int l = 0; l < L; ++l, ++lay) {
          for (int s = 0; s < 2; ++s) {
            for (int h = 0; h < NP; ++h) {
              // K-halves j0, j0 + 1 of piece h (for both streams): waited for by stream 0's step,
              // released after stream 1's
              const uint32_t j0 = (lay * NP + h) * 2;
              if (h == 0) {
                F3_T0();
                mbar_wait_cluster(&a_full[s], aph[s]);
                F3_ACC(ph_a);
                aph[s] ^= 1;
              }
              const uint32_t a_base = a_base0 + s * A_BYTES;
              for (int kh = 0; kh < 2; ++kh) {
                const uint32_t j = j0 + kh, b = j % NWB;
                if (s == 0) {
                  F3_T0();
                  mbar_wait_cluster(&w_full[b], (j / NWB) & 1);
                  F3_ACC(ph_w);
                }
                tc_fence_after();
                const uint32_t wb = w_base + b * WQ;
#pragma unroll 4
                for (int kk = 8 * kh; kk < 8 * kh + 8; ++kk) {
                  uint64_t ad = sdesc_sw128(a_base + (kk >> 2) * (128 * 128) + (kk & 3) * 32, 16, 1024);
                  uint64_t bd = sdesc_sw128(wb + ((kk >> 2) & 1) * (PR * 128) + (kk & 3) * 32, 16, 1024);
                  umma_bf16_pair(tmem + s * 256 + h * PN, ad, bd, idesc, kk > 0 ? 1u : 0u);
                }
                if (s == 1) umma_commit_pair(&w_free[b], 3);
              }
              if (h == NP - 1) umma_commit_pair(&acc_full[s], 3);
            }
          }
        }
      }
#ifdef DINR_PHASES
      if (p.dbg) {
        p.dbg[(size_t)blockIdx.x * 32 + 8] = ph_w;
        p.dbg[(size_t)blockIdx.x * 32 + 9] = ph_a;
      }
#endif
    }
  } else if (tid == 544) {
    // ============================================================ W loads (both CTAs)
    const uint8_t *wsrc = reinterpret_cast<const uint8_t *>(p.wpack);
    uint32_t lay = 0;
    [[maybe_unused]] unsigned long long ph_lf = 0;
    for (int64_t pi = cl; pi < n_iter; pi += ncl) {
      for (int l = 0; l < L; ++l, ++lay) {
        for (int h = 0; h < NP; ++h) {
          for (int kh = 0; kh < 2; ++kh) {
            const uint32_t j = (lay * NP + h) * 2 + kh, b = j % NWB;
            if (j >= NWB) {  // stream 1's MMAs on K-half j - NWB (this buffer's last use) retired
              F3_T0();
              mbar_wait_long(&w_free[b], ((j / NWB) - 1) & 1);
              F3_ACC(ph_lf);
            }
            uint64_t *bar = leader ? &w_full[b] : &w_loc[b];
            mbar_arrive_expect_tx(bar, WQ);
            // this CTA's rows [PN h + PR r, +PR) of 64-column K-blocks 2 kh, 2 kh + 1 of the W_l image
            for (int q = 0; q < 2; ++q)
              bulk_g2s(sW + b * WQ + q * (PR * 128),
                       wsrc + (size_t)l * W_LAYER + (2 * kh + q) * (H * 128) + (size_t)(PN * h + PR * rank) * 128,
                       PR * 128, bar);
          }
        }
      }
    }
#ifdef DINR_PHASES
    if (p.dbg) p.dbg[(size_t)blockIdx.x * 32 + 10] = ph_lf;
#endif
  } else if (tid == 608) {
    // ============================================================ peer: W halves landed -> leader
    // (a thread of its own, so the peer's loader keeps loads in flight like the leader's)
    if (!leader) {
      const uint32_t w_full_leader = mapa_shared(smem_u32(&w_full[0]), 0);
      uint32_t lay = 0;
      [[maybe_unused]] unsigned long long ph_ll = 0;
      for (int64_t pi = cl; pi < n_iter; pi += ncl)
        for (int l = 0; l < L; ++l, ++lay)
          for (uint32_t j = lay * NP * 2; j < (lay + 1) * NP * 2; ++j) {
            const uint32_t b = j % NWB;
            F3_T0();
            mbar_wait_long(&w_loc[b], (j / NWB) & 1);
            F3_ACC(ph_ll);
            mbar_arrive_remote(w_full_leader + b * 8);
          }
#ifdef DINR_PHASES
      if (p.dbg) p.dbg[(size_t)blockIdx.x * 32 + 11] = ph_ll;
#endif
    }
  } else if (tid == 576) {
    // ============================================================ h-stash stores (both CTAs)
    uint32_t rph[2] = {0, 0};
    [[maybe_unused]] unsigned long long ph_sa = 0, ph_sr = 0;
    for (int64_t pi = cl; pi < n_iter; pi += ncl) {
      for (int l = 0; l < L; ++l) {
        for (int s = 0; s < 2; ++s) {
          {
            F3_T0();
            mbar_wait_long(&a_rdy[s], rph[s]);
            F3_ACC(ph_sa);
          }
          rph[s] ^= 1;
          const int64_t tile = 4 * pi + 2 * s + rank;
          // layer l's input for the dW GEMM (l = 0: the GRFF features, unless the dW GEMM recomputes them)
          if (!p.zall && (l > 0 || p.stash_feat)) {
            STASH_S2G(p.hstash + ((size_t)l * p.n_tiles + tile) * A_BYTES, sA0 + s * A_BYTES, A_BYTES);
            bulk_commit();
            F3_T0();
            bulk_wait_read_all();
            F3_ACC(ph_sr);
          }
          mbar_arrive(&acc_full[s]);
        }
      }
    }
    bulk_wait_all();
#ifdef DINR_PHASES
    if (p.dbg) {
      p.dbg[(size_t)blockIdx.x * 32 + 12] = ph_sa;
      p.dbg[(size_t)blockIdx.x * 32 + 13] = ph_sr;
    }
#endif
  } else if (tid < 512) {
    // ============================================================ epilogue streams
    const int s = tid >> 8, wt = tid & 255;
    const int row = wt & 127, cg = wt >> 7;
    const uint32_t a_base = smem_u32(sA0) + s * A_BYTES;
    const uint32_t tmem_row = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(s * 256);
    const uint32_t a_full_leader = mapa_shared(smem_u32(&a_full[s]), 0);
    const uint64_t pol_z = policy_evict_first();
    uint32_t accph = 0;
    [[maybe_unused]] unsigned long long ph_e[4] = {0, 0, 0, 0};  // features, acc wait, layer epilogue, head sum
    auto hand_off = [&]() {  // A_s written (generic proxy) -> the pair MMA and this CTA's stash store
      fence_proxy_async_smem();
      asm volatile("bar.sync %0, 256;" ::"r"(1 + s) : "memory");
      if (wt == 0) {
        mbar_arrive(&a_rdy[s]);
        if (leader)
          mbar_arrive(&a_full[s]);
        else
          mbar_arrive_remote(a_full_leader);
      }
    };
    for (int64_t pi = cl; pi < n_iter; pi += ncl) {
      const int64_t tile = 4 * pi + 2 * s + rank;
      const int64_t g = tile * 128 + row;
      const bool valid = g < p.nsamp;
      // ---------------------------------------------------------------- a5/a6 features (as K2)
      {
        F3_T0();
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
        F3_ACC(ph_e[0]);
      }
      hand_off();
      // ---------------------------------------------------------------- a7/a8 layers
      float mu_acc = 0.f;
      for (int l = 0; l < L; ++l) {
        const bool last = (l == L - 1);
        {
          F3_T0();
          mbar_wait_long(&acc_full[s], accph);  // CTA scope: TMEM + own smem only
          F3_ACC(ph_e[1]);
        }
        accph ^= 1;
        tc_fence_after();
        F3_T0();
#pragma unroll 1
        for (int cb = cg * 4; cb < cg * 4 + 4; ++cb) {  // this thread's 32-column chunks
          uint32_t va[16], vb[16];  // both 16-column halves of the chunk in flight at once
          tmem_ld16(tmem_row + cb * 32, va);
          tmem_ld16(tmem_row + cb * 32 + 16, vb);
          tmem_wait_ld();
          reg_fence(va);
          reg_fence(vb);
#pragma unroll
          for (int q16 = 0; q16 < 2; ++q16) {
            const uint32_t(&v)[16] = q16 ? vb : va;
            const int col0 = cb * 32 + q16 * 16;
            // y = z / 2 (halved bias), t = tanh y: h = swish(z) = y (1 + t); sigma = (1 + t) / 2;
            // swish'(z) = sigma (1 + z (1 - sigma)) = sigma + sigma y (1 - t)
            float y[16], t[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              y[i] = fmaf(__uint_as_float(v[i]), 0.5f, sBias[l * H + col0 + i]);
              t[i] = tanh_approx(y[i]);
            }
            uint32_t s8[8];  // backward state, [16-column chunk][row][32 B] (the layout K3 reads)
            if (p.zall) {    // fp16 y of every layer
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                __half2 hh = __floats2half2_rn(y[2 * e], y[2 * e + 1]);
                s8[e] = *reinterpret_cast<uint32_t *>(&hh);
              }
            } else if (last) {  // fp16 z_{L-1} (= 2 y exactly)
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                __half2 hh = __floats2half2_rn(2.f * y[2 * e], 2.f * y[2 * e + 1]);
                s8[e] = *reinterpret_cast<uint32_t *>(&hh);
              }
            } else {  // bf16 swish'(z)
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const int i0 = 2 * e;
                const float s0 = fmaf(t[i0], 0.5f, 0.5f), s1 = fmaf(t[i0 + 1], 0.5f, 0.5f);
                s8[e] = pack_bf16x2(fmaf(s0, fmaf(-y[i0], t[i0], y[i0]), s0), fmaf(s1, fmaf(-y[i0 + 1], t[i0 + 1], y[i0 + 1]), s1));
              }
            }
            st_global_v8_hint(p.zstash + ((((size_t)l * p.n_tiles + tile) * (H / 16) + (col0 >> 4)) * 128 + row) * 32, s8,
                              pol_z);
            if (!last) {
              uint32_t w8[8];
#pragma unroll
              for (int e = 0; e < 8; ++e)
                w8[e] = pack_bf16x2(fmaf(y[2 * e], t[2 * e], y[2 * e]), fmaf(y[2 * e + 1], t[2 * e + 1], y[2 * e + 1]));
              st_shared_v4(a_base + sw128_offset(row, col0, 128), w8[0], w8[1], w8[2], w8[3]);
              st_shared_v4(a_base + sw128_offset(row, col0 + 8, 128), w8[4], w8[5], w8[6], w8[7]);
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i) mu_acc = fmaf(sWo[col0 + i], fmaf(y[i], t[i], y[i]), mu_acc);
            }
          }
        }
        tc_fence_before();
        if (!last) hand_off();
        F3_ACC(ph_e[2]);
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
#ifdef DINR_PHASES
      if (wt == 0 && p.dbg)
        for (int k = 0; k < 4; ++k) p.dbg[(size_t)blockIdx.x * 32 + s * 4 + k] = ph_e[k];
#endif
      // the last layer's A_s was not rewritten: the stash thread's arrival for it is still owed
      // (it stores inputs of layers 0 .. L-1 only), so nothing to hand off here
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // both CTAs done with the pair's TMEM
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 512);
  }
}

}  // namespace dinr
