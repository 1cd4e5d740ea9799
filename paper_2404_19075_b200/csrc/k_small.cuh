// k_small.cuh -- K4 loss/combine kernel, K5 weight pack, gradient assembly.
#pragma once
#include <cuda_bf16.h>

#include "internal.cuh"
#include "ptx_sm100.cuh"

namespace dinr {

// ---------------------------------------------------------------------------------------
// K5 weight pack: fp32 W_l ([out][in], D5 layout) -> bf16 SW128 K-major image per layer
// (rows = out, K = in; 64-column blocks of H rows x 128 B; 16-B chunk index ^= row % 8).
// The same image serves as the K-major B operand of the forward (N = out, K = in) and the
// MN-major B operand of the backward dX GEMM (N = in, K = out).
// ---------------------------------------------------------------------------------------
__global__ void k_pack_weights(const float *__restrict__ params, int H, int L, uint16_t *__restrict__ wpack,
                               uint16_t *__restrict__ wpack_half) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t per = (int64_t)H * H;
  if (q >= per * L) return;
  int l = (int)(q / per);
  int e = (int)(q - (int64_t)l * per);
  int o = e / H, i = e % H;
  float w = params[(int64_t)l * (per + H) + e];
  __nv_bfloat16 b = __float2bfloat16_rn(w);
  __nv_bfloat16 bh = __float2bfloat16_rn(0.5f * w);  // exact: a power-of-two scale of a bf16 value
  uint32_t off = sw128_offset((uint32_t)o, (uint32_t)i, (uint32_t)H) >> 1;
  wpack[(int64_t)l * per + off] = *reinterpret_cast<uint16_t *>(&b);
  wpack_half[(int64_t)l * per + off] = *reinterpret_cast<uint16_t *>(&bh);
}

// ---------------------------------------------------------------------------------------
// K4 combine + loss (one thread per pixel).
//   p_s   = wq_s * sum_c pchunk[ray s][c]    (eq:estforwmod with R7; pchunk = sums of M)
//   BEER  : m = min p_s, T = (1/S) sum e^{-(p_s-m)}, fhat = m - ln T    (eq:beerstransavg, R22)
//   LINEAR: fhat = (1/S) sum p_s                                         (eq:beersattenavg)
//   loss partial sum (y - fhat)^2 (eq:mainsqdist); upstream per ray for the raw head output
//   u_s = g pi_s wq_s mu0 with g = -2 (y - fhat)/n, pi_s = dfhat/dp_s (eq:partiald, R15).
// ---------------------------------------------------------------------------------------
constexpr int kLossThreads = 256;
constexpr int kMaxS = 16;

__global__ void __launch_bounds__(kLossThreads) k_loss(const float *__restrict__ wqa, const float *__restrict__ pchunk,
                                                       int S, int nc, int64_t n, const float *__restrict__ y,
                                                       int combine, float mu0, float *__restrict__ fhat,
                                                       float *__restrict__ p_sub, const float *__restrict__ I0,
                                                       float *__restrict__ Ihat, float *__restrict__ u,
                                                       float *__restrict__ loss_part) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  float r2 = 0.f;
  if (i < n) {
    float p[kMaxS], wq[kMaxS];
    for (int s = 0; s < S; ++s) {
      int64_t ray = i * S + s;
      wq[s] = wqa[ray];  // quadrature weight chord / N_s (K1's compact copy)
      float acc = 0.f;
      for (int c = 0; c < nc; ++c) acc += pchunk[ray * nc + c];
      p[s] = wq[s] > 0.f ? wq[s] * acc : 0.f;
      if (p_sub) p_sub[ray] = p[s];
    }
    float fh, T = 1.f, m = 0.f;
    if (combine == DINR_LINEAR) {
      float acc = 0.f;
      for (int s = 0; s < S; ++s) acc += p[s];
      fh = acc / (float)S;
    } else {
      m = p[0];
      for (int s = 1; s < S; ++s) m = fminf(m, p[s]);
      float acc = 0.f;
      for (int s = 0; s < S; ++s) acc += expf(-(p[s] - m));
      T = acc / (float)S;
      fh = m - logf(T);
    }
    if (fhat) fhat[i] = fh;
    if (Ihat) Ihat[i] = I0[i] * expf(-fh);
    if (y) {
      float res = y[i] - fh;
      r2 = res * res;
      float g = -2.f * res / (float)n;
      for (int s = 0; s < S; ++s) {
        float pi = combine == DINR_LINEAR ? 1.f / (float)S : expf(-(p[s] - m)) / ((float)S * T);
        u[i * S + s] = g * pi * wq[s] * mu0;
      }
    }
  }
  if (loss_part) {
    // deterministic block reduction
    __shared__ float red[kLossThreads / 32];
    for (int o = 16; o > 0; o >>= 1) r2 += __shfl_xor_sync(0xffffffffu, r2, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = r2;
    __syncthreads();
    if (threadIdx.x == 0) {
      float acc = 0.f;
      for (int w = 0; w < kLossThreads / 32; ++w) acc += red[w];
      loss_part[blockIdx.x] = acc;
    }
  }
}

// ---------------------------------------------------------------------------------------
// Gradient assembly: grad[q] (+)= sum over split partials in fixed order; grad[P] = loss.
// dw_part layout: [L][nmb][ksplit][128][H]; db_part: [L][nmb][ksplit][128];
// head_part: [nhead][H+1].
// ---------------------------------------------------------------------------------------
// db_part uses the split count ks_db (the zall path's bias partials come from K3's CTAs, the
// weight partials from the dW GEMM's K-split).
__global__ void k_assemble(int H, int L, int64_t P, int nmb, int ksplit, const float *__restrict__ dw_part,
                           const float *__restrict__ db_part, int ks_db, const float *__restrict__ head_part, int nhead,
                           const float *__restrict__ loss_part, int nloss, float inv_n, int accumulate,
                           float *__restrict__ grad) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q > P) return;
  float v = 0.f;
  int64_t per = (int64_t)H * H + H;
  if (q == P) {
    for (int b = 0; b < nloss; ++b) v += loss_part[b];
    v *= inv_n;
  } else if (q < (int64_t)L * per) {
    int l = (int)(q / per);
    int64_t e = q - (int64_t)l * per;
    if (e < (int64_t)H * H) {
      int o = (int)(e / H), i = (int)(e % H);
      int mb = o >> 7, ol = o & 127;
      const float *src = dw_part + ((((int64_t)l * nmb + mb) * ksplit) * 128 + ol) * H + i;
      for (int s = 0; s < ksplit; ++s) v += src[(int64_t)s * 128 * H];
    } else {
      int o = (int)(e - (int64_t)H * H);
      int mb = o >> 7, ol = o & 127;
      const float *src = db_part + (((int64_t)l * nmb + mb) * ks_db) * 128 + ol;
      for (int s = 0; s < ks_db; ++s) v += src[(int64_t)s * 128];
    }
  } else {
    int k = (int)(q - (int64_t)L * per);  // 0..H-1 -> w_o, H -> b_o
    for (int b = 0; b < nhead; ++b) v += head_part[(int64_t)b * (H + 1) + k];
  }
  grad[q] = accumulate ? grad[q] + v : v;
}

// N1: fused Adam step + re-pack of the bf16 weight images (one thread per parameter).
__global__ void k_adam_pack(float *__restrict__ params, const float *__restrict__ grad, float *__restrict__ m,
                            float *__restrict__ v, int64_t P, int H, int L, float lr, float b1, float b2, float eps,
                            float c1, float c2, float *__restrict__ ctx_params, uint16_t *__restrict__ wpack,
                            uint16_t *__restrict__ wpack_half) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= P) return;
  const float g = grad[q];
  const float mq = b1 * m[q] + (1.f - b1) * g;
  const float vq = b2 * v[q] + (1.f - b2) * g * g;
  m[q] = mq;
  v[q] = vq;
  const float w = params[q] - lr * (mq / c1) / (sqrtf(vq / c2) + eps);
  params[q] = w;
  ctx_params[q] = w;
  const int64_t per = (int64_t)H * H + H;
  // the bf16 SW128 images exist only for the BF16 path (H in {64,128,256}); FP32_VERIFY passes null
  if (wpack && q < (int64_t)L * per) {
    const int l = (int)(q / per);
    const int64_t e = q - (int64_t)l * per;
    if (e < (int64_t)H * H) {
      const int o = (int)(e / H), i = (int)(e % H);
      const uint32_t off = sw128_offset((uint32_t)o, (uint32_t)i, (uint32_t)H) >> 1;
      __nv_bfloat16 b = __float2bfloat16_rn(w), bh = __float2bfloat16_rn(0.5f * w);
      wpack[(int64_t)l * H * H + off] = *reinterpret_cast<uint16_t *>(&b);
      wpack_half[(int64_t)l * H * H + off] = *reinterpret_cast<uint16_t *>(&bh);
    }
  }
}

// Assembly for the fused path (H <= 128): layers [0, nu) from the dW GEMM partials
// ([l][ks5][128][H]), layers [nu, L) from the fused kernel's per-CTA TMEM partials
// ([l - nu][ksf][128][H]); fixed summation order -> deterministic.
// Gradient assembly for the fused path: parameter q sums its per-CTA / per-K-split partials.
// Block = 32 consecutive parameters (lanes, coalesced) x 8 warps; warp w sums partials w, w+8,
// ... and the 8 warp sums are added in fixed order (deterministic).
__global__ void __launch_bounds__(256) k_assemble2(int H, int L, int64_t P, int nu, int ks5,
                                                   const float *__restrict__ dw5, const float *__restrict__ db5, int ksf,
                                                   const float *__restrict__ dwf, const float *__restrict__ dbf,
                                                   const float *__restrict__ head_part, int nhead,
                                                   const float *__restrict__ loss_part, int nloss, float inv_n,
                                                   int accumulate, float *__restrict__ grad) {
  __shared__ float red[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t q = (int64_t)blockIdx.x * 32 + lane;
  const int64_t per = (int64_t)H * H + H;
  float v = 0.f;
  if (q == P) {
    for (int b = w; b < nloss; b += 8) v += loss_part[b];
  } else if (q < (int64_t)L * per) {
    const int l = (int)(q / per);
    const int64_t e = q - (int64_t)l * per;
    const bool f = l >= nu;
    const int ks = f ? ksf : ks5;
    const int ll = f ? l - nu : l;
    const float *src;
    size_t stride;
    if (e < (int64_t)H * H) {
      const int o = (int)(e / H), i = (int)(e % H);
      src = (f ? dwf : dw5) + ((size_t)ll * ks * 128 + o) * H + i;
      stride = (size_t)128 * H;
    } else {
      src = (f ? dbf : db5) + (size_t)ll * ks * 128 + (e - (int64_t)H * H);
      stride = 128;
    }
#pragma unroll 4
    for (int s = w; s < ks; s += 8) v += src[(size_t)s * stride];
  } else if (q < P) {
    const int k = (int)(q - (int64_t)L * per);
#pragma unroll 4
    for (int b = w; b < nhead; b += 8) v += head_part[(int64_t)b * (H + 1) + k];
  }
  red[w][lane] = v;
  __syncthreads();
  if (w == 0 && q <= P) {
    float t = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) t += red[j][lane];
    if (q == P) t *= inv_n;
    grad[q] = accumulate ? grad[q] + t : t;
  }
}

}  // namespace dinr
