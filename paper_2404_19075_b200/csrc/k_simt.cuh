// k_simt.cuh -- fp32 SIMT verification path (precision = DINR_FP32_VERIFY; the "K6 twins").
//
// Same math as the tensor-core path, staged through global memory with fp32 CUDA-core
// GEMMs and accurate sincospif/expf; meant for the 1e-5 projection parity mode, not speed.
//   features  h_0 = [cos 2 pi phi ; sin 2 pi phi], phi = B rbar
//   layers    z_l = W_l h_{l-1} + b_l, h_l = z_l sigma(z_l)
//   head      M = mu0 (w_o . h_L + b_o), ray chunks of 32 samples summed
//   backward  delta_l = e_l * swish'(z_l), dW_l = delta_l^T h_{l-1}, e_{l-1} = W_l^T delta_l
#pragma once
#include "internal.cuh"
#include "k_features.cuh"

namespace dinr {

__device__ __forceinline__ float sigmoid_acc(float z) { return 1.f / (1.f + expf(-z)); }

__global__ void s_features(const float4 *__restrict__ rec32, int64_t nsamp, int n_s, const float *__restrict__ B,
                           int C, float *__restrict__ h0, Jitter jit) {
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nsamp) return;
  int64_t ray = g / n_s;
  const uint32_t jr = (uint32_t)(g - ray * n_s);
  float jj = (float)jr + sample_offset(jit, ray, jr);
  float4 a = rec32[2 * ray], b = rec32[2 * ray + 1];
  float rb[4] = {a.w, a.z + jj * b.z, a.y + jj * b.y, a.x + jj * b.x};  // (t, z, y, x), R12
  float *out = h0 + g * (2 * C);
  for (int c = 0; c < C; ++c) {
    float phi = B[4 * c] * rb[0] + B[4 * c + 1] * rb[1] + B[4 * c + 2] * rb[2] + B[4 * c + 3] * rb[3];
    float sn, cs;
    sincospif(2.f * phi, &sn, &cs);
    out[c] = cs;
    out[C + c] = sn;
  }
}

// N4 voxels: GRFF features at the voxel centres (accurate sincospif, like s_features).
__global__ void s_vox_features(VoxGrid vg, int64_t n_vox, const float *__restrict__ B, int C, float *__restrict__ h0) {
  int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n_vox) return;
  bool inside;
  const float4 r = voxel_coords(vg, v, inside);
  const float rb[4] = {r.x, r.y, r.z, r.w};
  float *out = h0 + v * (2 * C);
  for (int c = 0; c < C; ++c) {
    float phi = B[4 * c] * rb[0] + B[4 * c + 1] * rb[1] + B[4 * c + 2] * rb[2] + B[4 * c + 3] * rb[3];
    float sn, cs;
    sincospif(2.f * phi, &sn, &cs);
    out[c] = cs;
    out[C + c] = sn;
  }
}

// C[m][n] = sum_k A(m,k) B(k,n), fp32, 64x64 tiles, BK = 16, 256 threads (4x4 per thread).
// mode 0: raw store to C at z*cz + (m>>7)*cmb + (m&127)*ldc + n (split-K partials, blockIdx.z)
// mode 1: + bias[n]; store Z[m*ldc+n] = z and Hout[m*ldc+n] = z sigma(z)
struct SgemmArgs {
  const float *A;
  int64_t sam, sak;
  const float *B;
  int64_t sbk, sbn;
  int64_t M, N, K, kchunk;
  int mode;
  float *C;
  int64_t ldc, cz, cmb;
  const float *bias;
  float *Z, *Hout;
};

__global__ void __launch_bounds__(256) s_gemm(SgemmArgs a) {
  __shared__ float As[16][64 + 4];
  __shared__ float Bs[16][64 + 4];
  int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  int64_t m0 = (int64_t)blockIdx.y * 64, n0 = (int64_t)blockIdx.x * 64;
  int64_t kb = (int64_t)blockIdx.z * a.kchunk, ke = min(a.K, kb + a.kchunk);
  float acc[4][4] = {};
  for (int64_t k0 = kb; k0 < ke; k0 += 16) {
    for (int e = threadIdx.x; e < 16 * 64; e += 256) {
      int kk = e / 64, mm = e % 64;
      int64_t k = k0 + kk;
      As[kk][mm] = (k < ke && m0 + mm < a.M) ? a.A[(m0 + mm) * a.sam + k * a.sak] : 0.f;
      Bs[kk][mm] = (k < ke && n0 + mm < a.N) ? a.B[k * a.sbk + (n0 + mm) * a.sbn] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        av[q] = As[kk][ty * 4 + q];
        bv[q] = Bs[kk][tx * 4 + q];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += av[i] * bv[j];
    }
    __syncthreads();
  }
  for (int i = 0; i < 4; ++i) {
    int64_t m = m0 + ty * 4 + i;
    if (m >= a.M) continue;
    for (int j = 0; j < 4; ++j) {
      int64_t nn = n0 + tx * 4 + j;
      if (nn >= a.N) continue;
      if (a.mode == 0) {
        a.C[blockIdx.z * a.cz + (m >> 7) * a.cmb + (m & 127) * a.ldc + nn] = acc[i][j];
      } else {
        float z = acc[i][j] + a.bias[nn];
        a.Z[m * a.ldc + nn] = z;
        a.Hout[m * a.ldc + nn] = z * sigmoid_acc(z);
      }
    }
  }
}

// Ray chunk sums of M = mu0 (w_o . h_L + b_o): one warp per 32 samples.
// mu per sample: 32-sample chunk sums into pchunk, or (smu != null: N_s not a multiple of 32) the
// per-sample values into smu for s_raysum
__global__ void s_head(const float *__restrict__ hL, int64_t nsamp, int H, const float *__restrict__ wo,
                       float mu0, float *__restrict__ pchunk, float *__restrict__ smu) {
  const float bo = wo[H];
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  float mu = 0.f;
  if (g < nsamp) {
    const float *h = hL + g * H;
    float acc = 0.f;
    for (int k = 0; k < H; ++k) acc += wo[k] * h[k];
    mu = mu0 * (acc + bo);
  }
  if (smu) {
    if (g < nsamp) smu[g] = mu;
    return;
  }
  for (int o = 16; o > 0; o >>= 1) mu += __shfl_xor_sync(0xffffffffu, mu, o);
  if ((threadIdx.x & 31) == 0 && g < nsamp) pchunk[g >> 5] = mu;
}

// per-ray sums of mu (fixed order), one ray per thread
__global__ void s_raysum(const float *__restrict__ smu, int64_t n_rays, int n_s, float *__restrict__ psum) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rays) return;
  float acc = 0.f;
  for (int j = 0; j < n_s; ++j) acc += smu[r * n_s + j];
  psum[r] = acc;
}

// N4 voxels: mu = mu0 (w_o . h_L + b_o) per voxel, 0 outside the FOV cylinder (R25).
__global__ void s_vox_head(VoxGrid vg, const float *__restrict__ hL, int64_t n_vox, int H, const float *__restrict__ wo,
                           float mu0, float *__restrict__ out) {
  int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n_vox) return;
  bool inside;
  (void)voxel_coords(vg, v, inside);
  const float *h = hL + v * H;
  float acc = 0.f;
  for (int k = 0; k < H; ++k) acc += wo[k] * h[k];
  out[v] = inside ? mu0 * (acc + wo[H]) : 0.f;
}

// delta = e * swish'(z), swish'(z) = sigma (1 + z (1 - sigma)); for the head layer
// e = u_ray * w_o (u from K4, per ray).
__global__ void s_delta(float *__restrict__ e, const float *__restrict__ z, int64_t nsamp, int H,
                        const float *__restrict__ u, int n_s, const float *__restrict__ wo) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nsamp * H) return;
  float zz = z[q];
  float sg = sigmoid_acc(zz);
  float ev = u ? u[(q / H) / n_s] * wo[q % H] : e[q];
  e[q] = ev * (sg * (1.f + zz * (1.f - sg)));
}

// Column sums over sample rows [z*rows_per, ...) with optional per-row weight u[row / n_s]:
// out[z*ostride + c] = sum_rows w_row X[row][c]; if wsum_out, out[z*ostride + H] = sum w.
__global__ void s_colsum(const float *__restrict__ X, int64_t nsamp, int H, int64_t rows_per,
                         const float *__restrict__ u, int n_s, float *__restrict__ out, int64_t ostride,
                         int64_t mbstride, int wsum_out) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  int z = blockIdx.y;
  if (c > H || (c == H && !wsum_out)) return;
  int64_t r0 = (int64_t)z * rows_per, r1 = min(nsamp, r0 + rows_per);
  float acc = 0.f;
  for (int64_t r = r0; r < r1; ++r) {
    float w = u ? u[r / n_s] : 1.f;
    acc += c < H ? w * X[r * H + c] : w;
  }
  if (c < H)
    out[(int64_t)z * ostride + (c >> 7) * mbstride + (c & 127)] = acc;
  else
    out[(int64_t)z * ostride + H] = acc;
}

}  // namespace dinr
