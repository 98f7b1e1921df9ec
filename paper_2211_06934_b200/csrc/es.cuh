// es.cuh -- zero-order ES estimator kernels.
//
// PAPER.md §2.2 "Zero-order Differentiation (ZD)": the gradient of
// the Gaussian smoothing f~(theta) = E[f(theta + sigma z)] is
// (1/sigma) E[f(theta + sigma z) z]. Two kernels:
//   es_perturb: rows theta +/- sigma z_i for the caller's black-box f;
//   es_grad:    g = c sum_i w_i z_i with w_i = f_i (naive) or
//               f_i^+ - f_i^- (antithetic), c = 1/(n sigma) or 1/(2 n sigma).
// The noise is never stored: z_ij is regenerated from a counter-based draw
// keyed on (seed, sample i, element pair k = j/2) (reading N3):
//   key_i = mix(seed ^ mix(i + golden)),  w = mix(key_i + k),
//   u1 = ((w >> 41) + .5) 2^-23,  u2 = ((w & 0x7FFFFF) + .5) 2^-23,
//   z_2k = sqrt(-2 ln u1) cos(2 pi u2), z_2k+1 = sqrt(-2 ln u1) sin(2 pi u2)
// (SplitMix64 finaliser `mix`; one draw per Box-Muller pair). u1, u2 are
// exact in fp32; log and sin/cos use the MUFU approximations (es_pair).
#pragma once
#include <stdint.h>

#include "vec.cuh"

namespace dopt {

constexpr int kEsMaxSamples = 4096;  // keys + weights staged in shared memory

__host__ __device__ __forceinline__ uint64_t es_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t es_key(uint64_t seed, int64_t i) {
  return es_mix(seed ^ es_mix((uint64_t)i + 0x9E3779B97F4A7C15ull));
}

// the Box-Muller pair (z_2k, z_2k+1)
__device__ __forceinline__ void es_pair(uint64_t key, int64_t k, float& z0, float& z1) {
  const uint64_t w = es_mix(key + (uint64_t)k);
  const float u1 = ((float)(uint32_t)(w >> 41) + 0.5f) * (1.0f / 8388608.0f);
  const float u2 = ((float)(uint32_t)(w & 0x7FFFFFull) + 0.5f) * (1.0f / 8388608.0f);
  // MUFU fast paths (the kernel is ALU-bound otherwise: 67% of HBM with the
  // accurate functions): lg2.approx for the log (rel. error ~2^-22),
  // sin/cos.approx on a = 2 pi (u2 - 1/2) in (-pi, pi) (abs. error ~2^-21),
  // with sin(2 pi u2) = -sin(a), cos(2 pi u2) = -cos(a) exactly.
  const float r = sqrtf(-2.0f * 0.69314718055994531f * __log2f(u1));
  const float a = 6.28318530717958648f * (u2 - 0.5f);
  z0 = -r * __cosf(a);
  z1 = -r * __sinf(a);
}

__device__ __forceinline__ float es_normal(uint64_t key, int64_t j) {
  float z0, z1;
  es_pair(key, j >> 1, z0, z1);
  return (j & 1) ? z1 : z0;
}

// the 4 draws of vector v (elements 4v .. 4v+3 = pairs 2v, 2v+1)
__device__ __forceinline__ void es_quad(uint64_t key, int64_t v, float (&z)[4]) {
  es_pair(key, 2 * v, z[0], z[1]);
  es_pair(key, 2 * v + 1, z[2], z[3]);
}

// out row r starts at r * ld (ld = numel rounded up to 4 elements, so every
// row is 16-byte aligned): naive r = i, antithetic r = 2i (+) and 2i+1 (-).
// Work item w = (vector v, sample group q): a thread computes samples
// [q*spg, (q+1)*spg) of vector v. Large trees use spg = n_samples (theta is
// read once, each warp writes coalesced rows); small trees split the samples
// so that the grid still fills the GPU.
__global__ void __launch_bounds__(256) es_perturb_kernel(int64_t numel, int64_t n_samples,
                                                         int64_t sample0, int antithetic,
                                                         float sigma, uint64_t seed,
                                                         int64_t spg,
                                                         const float* __restrict__ theta,
                                                         float* __restrict__ out) {
  extern __shared__ uint64_t s_es[];
  uint64_t* s_key = s_es;
  for (int64_t i = threadIdx.x; i < n_samples; i += blockDim.x) s_key[i] = es_key(seed, sample0 + i);
  __syncthreads();
  const int reps = antithetic ? 2 : 1;
  const int64_t ld = (numel + 3) & ~int64_t(3);
  const int64_t nvec = (numel + 3) >> 2;  // last vector may be partial
  const int64_t groups = (n_samples + spg - 1) / spg;
  const int64_t total = nvec * groups, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < total; w += stride) {
    const int64_t q = groups == 1 ? 0 : w / nvec;  // (no 64-bit division when unsplit)
    const int64_t v = w - q * nvec;
    const bool full = 4 * v + 4 <= numel;
    float th[4];
    if (full) {
      load4(theta, v, th);
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) th[e] = 4 * v + e < numel ? theta[4 * v + e] : 0.f;
    }
    const int64_t i1 = min(n_samples, (q + 1) * spg);
    for (int64_t i = q * spg; i < i1; ++i) {
      float z[4], p[4], m[4];
      es_quad(s_key[i], v, z);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float sz = sigma * z[e];
        p[e] = th[e] + sz;
        m[e] = th[e] - sz;
      }
      float* row = out + (i * reps) * ld;
      if (full) {
        store4(row, v, p);
        if (antithetic) store4(row + ld, v, m);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {  // constant indices: p, m stay in registers
          if (4 * v + e < numel) {
            row[4 * v + e] = p[e];
            if (antithetic) row[ld + 4 * v + e] = m[e];
          }
        }
      }
    }
  }
}

// grad[j] = scale * sum_i w_i z_ij. SPLIT = false: a thread owns a vector and
// loops over all samples (large trees). SPLIT = true: a warp owns a vector,
// lanes take samples lane, lane+32, ..., then a fixed-order xor-shuffle sum
// (small trees with many samples). Both fp64-accumulated, deterministic.
template <bool SPLIT>
__global__ void __launch_bounds__(256) es_grad_kernel(int64_t numel, int64_t n_samples,
                                                      int antithetic, double scale,
                                                      uint64_t seed,
                                                      const float* __restrict__ f,
                                                      float* __restrict__ grad) {
  extern __shared__ uint64_t s_es[];
  uint64_t* s_key = s_es;
  float* s_w = reinterpret_cast<float*>(s_es + n_samples);
  for (int64_t i = threadIdx.x; i < n_samples; i += blockDim.x) {
    s_key[i] = es_key(seed, i);
    s_w[i] = antithetic ? f[2 * i] - f[2 * i + 1] : f[i];
  }
  __syncthreads();
  const int64_t nvec = (numel + 3) >> 2;
  const int lanes = SPLIT ? 32 : 1;
  const int lane = SPLIT ? (threadIdx.x & 31) : 0;
  const int64_t stride = (int64_t)gridDim.x * (blockDim.x / lanes);
  for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / lanes; v < nvec; v += stride) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t i = lane; i < n_samples; i += lanes) {
      const float w = s_w[i];
      float z[4];
      es_quad(s_key[i], v, z);
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[e] += (double)(w * z[e]);
    }
    if (SPLIT) {
#pragma unroll
      for (int e = 0; e < 4; ++e)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
    }
    if (lane == 0) {
      const float o[4] = {(float)(acc[0] * scale), (float)(acc[1] * scale),
                          (float)(acc[2] * scale), (float)(acc[3] * scale)};
      if (4 * v + 4 <= numel) {
        store4(grad, v, o);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (4 * v + e < numel) grad[4 * v + e] = o[e];
      }
    }
  }
}

}  // namespace dopt
