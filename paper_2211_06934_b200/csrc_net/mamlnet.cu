// libmamlnet.so -- memory-bound layers of the task-batched MAML network (C4)
// for sm_100a. Contract and formulas: include/mamlnet.h; derivation of the
// norm/pool second derivative: DESIGN.md §8.
//
// Layout: activations [G, B, H, W] with G = T*C groups; every group's
// n = B*H*W elements are contiguous. The norm/pool kernels run one CTA per
// group (batch statistics are per group), two or three passes over the
// group: the first pass leaves the group's span in L2 for the next (a
// layer-1 query group is 235 KB; 148 SMs x a few CTAs stay well inside the
// 126 MB L2). Group sums are fp64 (exact squares of fp32 inputs; order fixed
// by the block-reduction tree, so results are bitwise reproducible).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <string>

#include "mamlnet.h"

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

int fail(const char* msg) {
  g_err = msg;
  return NET_EINVAL;
}

int launched() {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_err = cudaGetErrorString(e);
    return NET_ECUDA;
  }
  return NET_OK;
}

constexpr uint8_t kOff = 255;  // inactive window (ReLU off)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sum K doubles over the block (fixed tree order). sm: >= 32*K doubles.
template <int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double* sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) sm[warp * K + k] = v[k];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double s = lane < nw ? sm[lane * K + k] : 0.0;
      s = warp_sum(s);
      if (lane == 0) sm[32 * K + k] = s;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = sm[32 * K + k];
}

struct Geo {  // one group's geometry
  int B, H, W, HW, H2, W2, P2;  // P2 = H2*W2
  int n, np;                    // elements, pooled elements
  __device__ Geo(int B_, int H_, int W_) : B(B_), H(H_), W(W_) {
    HW = H * W;
    H2 = H >> 1;
    W2 = W >> 1;
    P2 = H2 * W2;
    n = B * HW;
    np = B * P2;
  }
  // flat element index of pooled p's window position k (0..3)
  __device__ __forceinline__ int elem(int p, int k) const {
    int b = p / P2, r = p - b * P2, y2 = r / W2, x2 = r - y2 * W2;
    return b * HW + (2 * y2 + (k >> 1)) * W + 2 * x2 + (k & 1);
  }
  // pooled index and window position of element i (-1 if outside every window)
  __device__ __forceinline__ int pooled(int i, int& k) const {
    int b = i / HW, r = i - b * HW, y = r / W, x = r - y * W;
    int y2 = y >> 1, x2 = x >> 1;
    if (y2 >= H2 || x2 >= W2) return -1;
    k = ((y & 1) << 1) | (x & 1);
    return b * P2 + y2 * W2 + x2;
  }
};

// ------------------------------------------------------------ im2col / col2im
__global__ void __launch_bounds__(256) im2col_kernel(int B, int H, int W, const float* __restrict__ h,
                                                     float* __restrict__ cols) {
  const int64_t gk = blockIdx.x;  // (group, tap)
  const int g = (int)(gk / 9), k = (int)(gk - (int64_t)g * 9);
  const int di = k / 3 - 1, dj = k % 3 - 1;
  const int HW = H * W, n = B * HW;
  const float* src = h + (int64_t)g * n;
  float* dst = cols + gk * n;
  for (int i = blockIdx.y * blockDim.x + threadIdx.x; i < n; i += gridDim.y * blockDim.x) {
    int b = i / HW, r = i - b * HW, y = r / W, x = r - y * W;
    int ys = y + di, xs = x + dj;
    float v = 0.f;
    if ((unsigned)ys < (unsigned)H && (unsigned)xs < (unsigned)W) v = __ldg(src + b * HW + ys * W + xs);
    __stcs(dst + i, v);
  }
}

__global__ void __launch_bounds__(256) col2im_kernel(int B, int H, int W, const float* __restrict__ cols,
                                                     float* __restrict__ dh) {
  const int64_t g = blockIdx.x;
  const int HW = H * W, n = B * HW;
  const float* src = cols + g * 9 * (int64_t)n;
  float* dst = dh + g * n;
  for (int i = blockIdx.y * blockDim.x + threadIdx.x; i < n; i += gridDim.y * blockDim.x) {
    int b = i / HW, r = i - b * HW, y = r / W, x = r - y * W;
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      int ys = y - (k / 3 - 1), xs = x - (k % 3 - 1);
      if ((unsigned)ys < (unsigned)H && (unsigned)xs < (unsigned)W)
        s += __ldcs(src + (int64_t)k * n + b * HW + ys * W + xs);
    }
    dst[i] = s;
  }
}

// ----------------------------------------------------- batch norm + pool + relu
__global__ void bnpool_fwd_kernel(int B, int H, int W, const float* __restrict__ x,
                                  const float* __restrict__ gamma, const float* __restrict__ beta,
                                  double eps, float* __restrict__ out, uint8_t* __restrict__ code,
                                  float* __restrict__ mean_out, float* __restrict__ rstd_out) {
  __shared__ double sm[32 * 2 + 2];
  const Geo q(B, H, W);
  const int64_t g = blockIdx.x;
  const float* xg = x + g * q.n;
  double v[2] = {0.0, 0.0};
  for (int i = threadIdx.x; i < q.n; i += blockDim.x) {
    double a = (double)xg[i];
    v[0] += a;
    v[1] += a * a;
  }
  block_sum<2>(v, sm);
  const double mu = v[0] / q.n;
  double var = v[1] / q.n - mu * mu;
  var = var > 0.0 ? var : 0.0;
  const double rd = 1.0 / sqrt(var + eps);
  const float m = (float)mu, r = (float)rd, ga = gamma[g], be = beta[g];
  if (threadIdx.x == 0) {
    mean_out[g] = m;
    rstd_out[g] = r;
  }
  const float s = ga * r;  // z = s*(x - m) + be
  float* og = out + g * q.np;
  uint8_t* cg = code + g * q.np;
  for (int p = threadIdx.x; p < q.np; p += blockDim.x) {
    const int e0 = q.elem(p, 0);
    float best = s * (xg[e0] - m) + be;
    int kb = 0;
    float z1 = s * (xg[e0 + 1] - m) + be;
    if (z1 > best) best = z1, kb = 1;
    float z2 = s * (xg[e0 + W] - m) + be;
    if (z2 > best) best = z2, kb = 2;
    float z3 = s * (xg[e0 + W + 1] - m) + be;
    if (z3 > best) best = z3, kb = 3;
    const bool on = best > 0.f;
    og[p] = on ? best : 0.f;
    cg[p] = on ? (uint8_t)kb : kOff;
  }
}

// dy of element i (the pooled cotangent routed to the window maximum)
__device__ __forceinline__ float routed(const Geo& q, int i, const float* __restrict__ dpg,
                                        const uint8_t* __restrict__ cg) {
  int k;
  const int p = q.pooled(i, k);
  if (p < 0) return 0.f;
  return cg[p] == k ? dpg[p] : 0.f;
}

__global__ void bnpool_bwd_kernel(int B, int H, int W, const float* __restrict__ dp,
                                  const uint8_t* __restrict__ code, const float* __restrict__ x,
                                  const float* __restrict__ gamma, const float* __restrict__ mean,
                                  const float* __restrict__ rstd, float* __restrict__ dx,
                                  float* __restrict__ dgamma, float* __restrict__ dbeta) {
  __shared__ double sm[32 * 2 + 2];
  const Geo q(B, H, W);
  const int64_t g = blockIdx.x;
  const float* xg = x + g * q.n;
  const float* dpg = dp + g * q.np;
  const uint8_t* cg = code + g * q.np;
  const float m = mean[g], r = rstd[g];
  double v[2] = {0.0, 0.0};
  for (int p = threadIdx.x; p < q.np; p += blockDim.x) {
    const uint8_t c = cg[p];
    if (c != kOff) {
      const float d = dpg[p];
      const float xh = (xg[q.elem(p, c)] - m) * r;
      v[0] += (double)d;
      v[1] += (double)d * (double)xh;
    }
  }
  block_sum<2>(v, sm);
  if (threadIdx.x == 0) {
    dbeta[g] = (float)v[0];
    dgamma[g] = (float)v[1];
  }
  const float A = (float)(v[0] / q.n), Bm = (float)(v[1] / q.n), c0 = gamma[g] * r;
  float* dxg = dx + g * q.n;
  for (int i = threadIdx.x; i < q.n; i += blockDim.x) {
    const float xh = (xg[i] - m) * r;
    const float dy = routed(q, i, dpg, cg);
    dxg[i] = c0 * (dy - A - xh * Bm);
  }
}

__global__ void bnpool_bwd2_kernel(int B, int H, int W, const float* __restrict__ gdx,
                                   const float* __restrict__ gdgamma, const float* __restrict__ gdbeta,
                                   const float* __restrict__ dp, const uint8_t* __restrict__ code,
                                   const float* __restrict__ x, const float* __restrict__ gamma,
                                   const float* __restrict__ mean, const float* __restrict__ rstd,
                                   const float* __restrict__ dgamma, const float* __restrict__ dbeta,
                                   float* __restrict__ g_dp, float* __restrict__ g_x,
                                   float* __restrict__ g_gamma) {
  __shared__ double sm[32 * 3 + 3];
  const Geo q(B, H, W);
  const int64_t g = blockIdx.x;
  const float* xg = x + g * q.n;
  const float* dpg = dp + g * q.np;
  const uint8_t* cg = code + g * q.np;
  const float* gg = gdx ? gdx + g * q.n : nullptr;
  const float m = mean[g], r = rstd[g], ga = gamma[g];
  const float gdg = gdgamma ? gdgamma[g] : 0.f, gdb = gdbeta ? gdbeta[g] : 0.f;
  const double nd = (double)q.n;
  // sums: G1 = sum gdx, Gx = sum gdx*xh, Gd = sum gdx*dy
  double v[3] = {0.0, 0.0, 0.0};
  if (gg) {
    for (int i = threadIdx.x; i < q.n; i += blockDim.x) {
      const float t = gg[i];
      v[0] += (double)t;
      v[1] += (double)t * (double)((xg[i] - m) * r);
    }
    for (int p = threadIdx.x; p < q.np; p += blockDim.x) {
      const uint8_t c = cg[p];
      if (c != kOff) v[2] += (double)dpg[p] * (double)gg[q.elem(p, c)];
    }
  }
  block_sum<3>(v, sm);
  const double A = (double)dbeta[g] / nd, Bm = (double)dgamma[g] / nd;
  const double G1 = v[0], Gx = v[1], GD = v[2] - A * G1;
  const double gr = (double)ga * (double)r;
  if (threadIdx.x == 0) g_gamma[g] = (float)((double)r * (GD - Bm * Gx));
  // h = -gr*(dy*Gx/n + Bm*gdx) + gdg*dy = dy*ch + gdx*cg_
  const double mean_h = -gr * (A * Gx + Bm * G1) / nd + gdg * A;
  const double mean_hx = -2.0 * gr * Bm * Gx / nd + gdg * Bm;
  const double kx = gr * (double)r * (GD - Bm * Gx) / nd;
  const float ch = (float)(-gr * Gx / nd + gdg), cgd = (float)(-gr * Bm);
  const float mh = (float)mean_h, mhx = (float)mean_hx, fkx = (float)kx;
  float* gxg = g_x + g * q.n;
  for (int i = threadIdx.x; i < q.n; i += blockDim.x) {
    const float xh = (xg[i] - m) * r;
    const float dy = routed(q, i, dpg, cg);
    const float t = gg ? gg[i] : 0.f;
    const float h = dy * ch + t * cgd;
    gxg[i] = r * (h - mh - xh * mhx) - fkx * xh;
  }
  // g_dy = gr*(gdx - G1/n - xh*Gx/n) + gdg*xh + gdb at the routed positions
  const float fgr = (float)gr, g1n = (float)(G1 / nd), gxn = (float)(Gx / nd);
  float* gdpg = g_dp + g * q.np;
  for (int p = threadIdx.x; p < q.np; p += blockDim.x) {
    const uint8_t c = cg[p];
    float o = 0.f;
    if (c != kOff) {
      const int e = q.elem(p, c);
      const float xh = (xg[e] - m) * r;
      const float t = gg ? gg[e] : 0.f;
      o = fgr * (t - g1n - xh * gxn) + gdg * xh + gdb;
    }
    gdpg[p] = o;
  }
}

bool geo_ok(int64_t G, int64_t B, int64_t H, int64_t W, bool pool) {
  if (G < 0 || B < 1 || H < 1 || W < 1) return false;
  if (pool && (H < 2 || W < 2)) return false;
  if (B * H * W > (int64_t)1 << 30) return false;
  return G < ((int64_t)1 << 31) / 9;
}

int threads_for(int64_t n) { return n >= 16384 ? 512 : 256; }

dim3 stream_grid(int64_t rows, int64_t n) {
  // enough blocks to fill 148 SMs x 8 resident blocks; each loops inside its row
  int64_t chunks = (148 * 8 + rows - 1) / rows, most = (n + 255) / 256;
  if (chunks > most) chunks = most;
  if (chunks > 65535) chunks = 65535;
  if (chunks < 1) chunks = 1;
  return dim3((unsigned)rows, (unsigned)chunks);
}

}  // namespace

extern "C" {

int net_im2col3x3(int64_t G, int64_t B, int64_t H, int64_t W, const float* h, float* cols,
                  void* stream) {
  if (!geo_ok(G, B, H, W, false)) return fail("net_im2col3x3: bad geometry");
  if (G == 0) return NET_OK;
  if (!h || !cols) return fail("net_im2col3x3: NULL pointer");
  im2col_kernel<<<stream_grid(G * 9, B * H * W), 256, 0, (cudaStream_t)stream>>>(
      (int)B, (int)H, (int)W, h, cols);
  return launched();
}

int net_col2im3x3(int64_t G, int64_t B, int64_t H, int64_t W, const float* cols, float* dh,
                  void* stream) {
  if (!geo_ok(G, B, H, W, false)) return fail("net_col2im3x3: bad geometry");
  if (G == 0) return NET_OK;
  if (!cols || !dh) return fail("net_col2im3x3: NULL pointer");
  col2im_kernel<<<stream_grid(G, B * H * W), 256, 0, (cudaStream_t)stream>>>(
      (int)B, (int)H, (int)W, cols, dh);
  return launched();
}

int net_bnpool_fwd(int64_t G, int64_t B, int64_t H, int64_t W, const float* x,
                   const float* gamma, const float* beta, double eps, float* out, uint8_t* code,
                   float* mean, float* rstd, void* stream) {
  if (!geo_ok(G, B, H, W, true)) return fail("net_bnpool_fwd: bad geometry");
  if (!(eps >= 0.0)) return fail("net_bnpool_fwd: eps must be >= 0");
  if (G == 0) return NET_OK;
  if (!x || !gamma || !beta || !out || !code || !mean || !rstd)
    return fail("net_bnpool_fwd: NULL pointer");
  bnpool_fwd_kernel<<<(unsigned)G, threads_for(B * H * W), 0, (cudaStream_t)stream>>>(
      (int)B, (int)H, (int)W, x, gamma, beta, eps, out, code, mean, rstd);
  return launched();
}

int net_bnpool_bwd(int64_t G, int64_t B, int64_t H, int64_t W, const float* dp,
                   const uint8_t* code, const float* x, const float* gamma, const float* mean,
                   const float* rstd, float* dx, float* dgamma, float* dbeta, void* stream) {
  if (!geo_ok(G, B, H, W, true)) return fail("net_bnpool_bwd: bad geometry");
  if (G == 0) return NET_OK;
  if (!dp || !code || !x || !gamma || !mean || !rstd || !dx || !dgamma || !dbeta)
    return fail("net_bnpool_bwd: NULL pointer");
  bnpool_bwd_kernel<<<(unsigned)G, threads_for(B * H * W), 0, (cudaStream_t)stream>>>(
      (int)B, (int)H, (int)W, dp, code, x, gamma, mean, rstd, dx, dgamma, dbeta);
  return launched();
}

int net_bnpool_bwd2(int64_t G, int64_t B, int64_t H, int64_t W, const float* gdx,
                    const float* gdgamma, const float* gdbeta, const float* dp,
                    const uint8_t* code, const float* x, const float* gamma, const float* mean,
                    const float* rstd, const float* dgamma, const float* dbeta, float* g_dp,
                    float* g_x, float* g_gamma, void* stream) {
  if (!geo_ok(G, B, H, W, true)) return fail("net_bnpool_bwd2: bad geometry");
  if (G == 0) return NET_OK;
  if (!dp || !code || !x || !gamma || !mean || !rstd || !dgamma || !dbeta || !g_dp || !g_x ||
      !g_gamma)
    return fail("net_bnpool_bwd2: NULL pointer");
  bnpool_bwd2_kernel<<<(unsigned)G, threads_for(B * H * W), 0, (cudaStream_t)stream>>>(
      (int)B, (int)H, (int)W, gdx, gdgamma, gdbeta, dp, code, x, gamma, mean, rstd, dgamma,
      dbeta, g_dp, g_x, g_gamma);
  return launched();
}

const char* net_last_error(void) { return g_err.c_str(); }
int net_abi_version(void) { return MAMLNET_ABI_VERSION; }
int64_t net_launch_count(void) { return g_launches.load(); }

}  // extern "C"
