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
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stddef.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "mamlnet.h"

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

int fail(const char* msg) {
  g_err = msg;
  return NET_EINVAL;
}
int fail(const std::string& msg) { return fail(msg.c_str()); }

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

// Division by a per-launch constant d as a multiply-high: q = umulhi(i, m)
// with m = ceil(2^32 / d) is exact whenever i * d < 2^32 (the rounding error
// i*(m*d - 2^32)/(d*2^32) stays below 1/d); otherwise plain division.
struct FastDiv {
  uint32_t d, m;
  bool fast;
  __device__ FastDiv() : d(1), m(0), fast(false) {}
  __device__ FastDiv(uint32_t d_, uint32_t limit) : d(d_ > 0 ? d_ : 1) {
    fast = d > 1 && (uint64_t)limit * d < (1ull << 32);
    m = d > 1 ? (uint32_t)(((1ull << 32) + d - 1) / d) : 0u;
  }
  __device__ __forceinline__ uint32_t div(uint32_t i) const {
    return d == 1 ? i : (fast ? __umulhi(i, m) : i / d);
  }
};

struct Geo {  // one group's geometry
  int B, H, W, HW, H2, W2, P2;  // P2 = H2*W2
  int n, np;                    // elements, pooled elements
  int L, nl, lw;                // leftover elements (outside every window) per image, total,
                                // of which the odd last column contributes lw per image
  FastDiv dHW, dW, dP2, dW2, dL;
  __device__ Geo(int B_, int H_, int W_) : B(B_), H(H_), W(W_) {
    HW = H * W;
    H2 = H >> 1;
    W2 = W >> 1;
    P2 = H2 * W2;
    n = B * HW;
    np = B * P2;
    lw = (W & 1) ? 2 * H2 : 0;
    L = lw + ((H & 1) ? W : 0);
    nl = B * L;
    dHW = FastDiv(HW, n);
    dW = FastDiv(W, n);
    dP2 = FastDiv(P2 > 0 ? P2 : 1, n);
    dW2 = FastDiv(W2 > 0 ? W2 : 1, n);
    dL = FastDiv(L > 0 ? L : 1, n);
  }
  // flat element index of pooled p's window position 0; position k adds off(k)
  __device__ __forceinline__ int elem0(int p) const {
    const int b = (int)dP2.div(p), r = p - b * P2, y2 = (int)dW2.div(r), x2 = r - y2 * W2;
    return b * HW + 2 * y2 * W + 2 * x2;
  }
  __device__ __forceinline__ int off(int k) const { return (k >> 1) * W + (k & 1); }
  // Pooled value o at pooled index p written into the 3x3 / padding-1 im2col
  // of the pooled map (cols9 = this group's [9, B, H2, W2] block): tap (i, j)
  // of output position (y2-i+1, x2-j+1) reads source (y2, x2). Positions
  // whose source lies outside the map are not written (kept zero by the caller).
  __device__ __forceinline__ void scatter_cols(float* __restrict__ cols9, int p, float o) const {
    const int b = (int)dP2.div(p), r = p - b * P2, y2 = (int)dW2.div(r), x2 = r - y2 * W2;
    float* base = cols9 + b * P2;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const int y = y2 - i + 1;
      if ((unsigned)y >= (unsigned)H2) continue;
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int x = x2 - j + 1;
        if ((unsigned)x >= (unsigned)W2) continue;
        __stcs(base + (int64_t)(3 * i + j) * np + y * W2 + x, o);
      }
    }
  }
  // j-th element outside every window (odd last column, then odd last row)
  __device__ __forceinline__ int left(int j) const {
    const int b = (int)dL.div(j), r = j - b * L;
    return b * HW + (r < lw ? r * W + (W - 1) : (H - 1) * W + (r - lw));
  }
};

// ------------------------------------------------------------ im2col / col2im
// One thread per source position (b, y, x) of a group: the 9 taps of the
// output column are written from one index decode (coalesced per tap plane).
__global__ void __launch_bounds__(256) im2col_kernel(int B, int H, int W, const float* __restrict__ h,
                                                     float* __restrict__ cols) {
  const int64_t g = blockIdx.x;
  const int HW = H * W, n = B * HW;
  const FastDiv dHW(HW, n), dW(W, n);
  const float* src = h + g * n;
  float* dst = cols + g * 9 * (int64_t)n;
  for (int i = blockIdx.y * blockDim.x + threadIdx.x; i < n; i += gridDim.y * blockDim.x) {
    const int b = (int)dHW.div(i), r = i - b * HW, y = (int)dW.div(r), x = r - y * W;
    const float* row = src + b * HW;
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const int ys = y + k / 3 - 1, xs = x + k % 3 - 1;
      float v = 0.f;
      if ((unsigned)ys < (unsigned)H && (unsigned)xs < (unsigned)W) v = __ldg(row + ys * W + xs);
      __stcs(dst + (int64_t)k * n + i, v);
    }
  }
}

// im2col with 4 consecutive source positions per thread, 9 float4 stores (n % 4 == 0:
// every tap plane and the group base stay 16-byte aligned); the position is
// decoded once and stepped along the row.
__global__ void __launch_bounds__(256) im2col4_kernel(int B, int H, int W, const float* __restrict__ h,
                                                      float* __restrict__ cols) {
  const int64_t g = blockIdx.x;
  const int HW = H * W, n = B * HW, n4 = n >> 2;
  const FastDiv dHW(HW, n), dW(W, n);
  const float* src = h + g * n;
  float* dst = cols + g * 9 * (int64_t)n;
  for (int i4 = blockIdx.y * blockDim.x + threadIdx.x; i4 < n4; i4 += gridDim.y * blockDim.x) {
    const int i = i4 << 2;
    int b = (int)dHW.div(i), r = i - b * HW, y = (int)dW.div(r), x = r - y * W;
    float v[9][4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float* row = src + b * HW;
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        const int ys = y + k / 3 - 1, xs = x + k % 3 - 1;
        v[k][j] = ((unsigned)ys < (unsigned)H && (unsigned)xs < (unsigned)W) ? __ldg(row + ys * W + xs) : 0.f;
      }
      if (++x == W) {
        x = 0;
        if (++y == H) y = 0, ++b;
      }
    }
#pragma unroll
    for (int k = 0; k < 9; ++k)
      __stcs(reinterpret_cast<float4*>(dst + (int64_t)k * n + i), make_float4(v[k][0], v[k][1], v[k][2], v[k][3]));
  }
}

__global__ void __launch_bounds__(256) col2im_kernel(int B, int H, int W, const float* __restrict__ cols,
                                                     float* __restrict__ dh) {
  const int64_t g = blockIdx.x;
  const int HW = H * W, n = B * HW;
  const FastDiv dHW(HW, n), dW(W, n);
  const float* src = cols + g * 9 * (int64_t)n;
  float* dst = dh + g * n;
  for (int i = blockIdx.y * blockDim.x + threadIdx.x; i < n; i += gridDim.y * blockDim.x) {
    const int b = (int)dHW.div(i), r = i - b * HW, y = (int)dW.div(r), x = r - y * W;
    float v[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const int ys = y - (k / 3 - 1), xs = x - (k % 3 - 1);
      v[k] = ((unsigned)ys < (unsigned)H && (unsigned)xs < (unsigned)W)
                 ? __ldcs(src + (int64_t)k * n + b * HW + ys * W + xs)
                 : 0.f;
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 9; ++k) s += v[k];
    dst[i] = s;
  }
}

// ----------------------------------------------------- batch norm + pool + relu
// One group (task, channel) per thread-block CLUSTER of kc CTAs (kc = 1..8,
// chosen from the group count so that small task batches still fill the
// 148 SMs): CTA rank r owns the r-th slice of the group's elements and of its
// pooled elements; group sums are combined across the cluster through
// distributed shared memory, in rank order (identical in every CTA,
// bitwise reproducible for a given kc).
struct Slice {
  int lo, hi;
  __device__ Slice(int n, int r, int k) {
    lo = (int)((int64_t)n * r / k);
    hi = (int)((int64_t)n * (r + 1) / k);
  }
};

// Sum K doubles over the cluster: block tree, then the kc block totals in
// rank order through DSMEM. sm >= 32*K + K doubles; part >= K doubles.
template <int K>
__device__ __forceinline__ void cluster_sum(double (&v)[K], double* sm, double* part) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  block_sum<K>(v, sm);
  const unsigned kc = cl.num_blocks();
  if (kc == 1) return;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) part[k] = v[k];
  }
  cl.sync();
  if (threadIdx.x < K) {
    double t = 0.0;
    for (unsigned r = 0; r < kc; ++r) t += cl.map_shared_rank(part, r)[threadIdx.x];
    sm[32 * K + threadIdx.x] = t;
  }
  cl.sync();  // every CTA has read every part; none exits while still being read
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = sm[32 * K + k];
}

__global__ void __launch_bounds__(256, 6) bnpool_fwd_kernel(int B, int H, int W, const float* __restrict__ x,
                                  const float* __restrict__ gamma, const float* __restrict__ beta,
                                  double eps, float* __restrict__ out, uint8_t* __restrict__ code,
                                  float* __restrict__ mean_out, float* __restrict__ rstd_out,
                                  float* __restrict__ cols) {
  __shared__ double sm[32 * 2 + 2];
  __shared__ double part[2];
  const Geo q(B, H, W);
  const int kc = (int)cooperative_groups::this_cluster().num_blocks();
  const int rank = (int)cooperative_groups::this_cluster().block_rank();
  const int64_t g = blockIdx.x / kc;
  const float* xg = x + g * q.n;
  const Slice es(q.n, rank, kc), ps(q.np, rank, kc);
  double v[2] = {0.0, 0.0};
  for (int i = es.lo + threadIdx.x; i < es.hi; i += blockDim.x) {
    double a = (double)xg[i];
    v[0] += a;
    v[1] += a * a;
  }
  cluster_sum<2>(v, sm, part);
  const double mu = v[0] / q.n;
  double var = v[1] / q.n - mu * mu;
  var = var > 0.0 ? var : 0.0;
  const double rd = 1.0 / sqrt(var + eps);
  const float m = (float)mu, r = (float)rd, ga = gamma[g], be = beta[g];
  if (threadIdx.x == 0 && rank == 0) {
    mean_out[g] = m;
    rstd_out[g] = r;
  }
  const float s = ga * r;  // z = s*(x - m) + be
  float* og = out + g * q.np;
  uint8_t* cg = code + g * q.np;
  float* c9 = cols ? cols + g * 9 * (int64_t)q.np : nullptr;
  for (int p = ps.lo + threadIdx.x; p < ps.hi; p += blockDim.x) {
    const int e0 = q.elem0(p);
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
    if (c9) q.scatter_cols(c9, p, on ? best : 0.f);
  }
}

template <bool EVEN>  // W even: each window's two rows as float2 pairs (8-byte aligned)
__global__ void __launch_bounds__(256, EVEN ? 6 : 8) bnpool_bwd_kernel(int B, int H, int W, const float* __restrict__ dp,
                                  const uint8_t* __restrict__ code, const float* __restrict__ x,
                                  const float* __restrict__ gamma, const float* __restrict__ mean,
                                  const float* __restrict__ rstd, float* __restrict__ dx,
                                  float* __restrict__ dgamma, float* __restrict__ dbeta) {
  __shared__ double sm[32 * 2 + 2];
  __shared__ double part[2];
  const Geo q(B, H, W);
  const int kc = (int)cooperative_groups::this_cluster().num_blocks();
  const int rank = (int)cooperative_groups::this_cluster().block_rank();
  const int64_t g = blockIdx.x / kc;
  const Slice ps(q.np, rank, kc);
  const float* xg = x + g * q.n;
  const float* dpg = dp + g * q.np;
  const uint8_t* cg = code + g * q.np;
  const float m = mean[g], r = rstd[g];
  double v[2] = {0.0, 0.0};
  for (int p = ps.lo + threadIdx.x; p < ps.hi; p += blockDim.x) {
    const uint8_t c = cg[p];
    const float d = dpg[p];  // unconditional: only the x gather depends on the code
    if (c != kOff) {
      const float xh = (xg[q.elem0(p) + q.off(c)] - m) * r;
      v[0] += (double)d;
      v[1] += (double)d * (double)xh;
    }
  }
  cluster_sum<2>(v, sm, part);
  if (threadIdx.x == 0 && rank == 0) {
    dbeta[g] = (float)v[0];
    dgamma[g] = (float)v[1];
  }
  const float A = (float)(v[0] / q.n), Bm = (float)(v[1] / q.n), c0 = gamma[g] * r;
  float* dxg = dx + g * q.n;
  // dx over the windows (dy = dp at the window's code position, else 0) ...
  for (int p = ps.lo + threadIdx.x; p < ps.hi; p += blockDim.x) {
    const int e0 = q.elem0(p);
    const uint8_t c = cg[p];
    const float dl = dpg[p], d = c != kOff ? dl : 0.f;  // unconditional load
    if constexpr (EVEN) {
      const float2 t = *reinterpret_cast<const float2*>(xg + e0);
      const float2 u = *reinterpret_cast<const float2*>(xg + e0 + W);
      const float xv[4] = {t.x, t.y, u.x, u.y};
      float o[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) o[k] = c0 * ((c == k ? d : 0.f) - A - (xv[k] - m) * r * Bm);
      *reinterpret_cast<float2*>(dxg + e0) = make_float2(o[0], o[1]);
      *reinterpret_cast<float2*>(dxg + e0 + W) = make_float2(o[2], o[3]);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int e = e0 + q.off(k);
        const float xh = (xg[e] - m) * r;
        dxg[e] = c0 * ((c == k ? d : 0.f) - A - xh * Bm);
      }
    }
  }
  // ... and over the elements outside every window (dy = 0)
  const Slice ls(q.nl, rank, kc);
  for (int j = ls.lo + threadIdx.x; j < ls.hi; j += blockDim.x) {
    const int e = q.left(j);
    dxg[e] = c0 * (-A - (xg[e] - m) * r * Bm);
  }
}

// MINB: 8 resident blocks for per-CTA slices of 2K-8K elements, else 6 (8 is
// faster on the 4.9K-element slices -- 14x14 at 32 tasks, 28x28 at 4 --
// slower on the 28x28 layer's 9.8K slices at 32 tasks and on the 7x7
// layer's 1.2K: profiles/r01f_bn_minblocks_sweep.txt, r01f_bn_bwd2_minb.txt)
template <int MINB>
__global__ void __launch_bounds__(256, MINB) bnpool_bwd2_kernel(int B, int H, int W, const float* __restrict__ gdx,
                                   const float* __restrict__ gdgamma, const float* __restrict__ gdbeta,
                                   const float* __restrict__ dp, const uint8_t* __restrict__ code,
                                   const float* __restrict__ x, const float* __restrict__ gamma,
                                   const float* __restrict__ mean, const float* __restrict__ rstd,
                                   const float* __restrict__ dgamma, const float* __restrict__ dbeta,
                                   float* __restrict__ g_dp, float* __restrict__ g_x,
                                   float* __restrict__ g_gamma) {
  __shared__ double sm[32 * 3 + 3];
  __shared__ double part[3];
  const Geo q(B, H, W);
  const int kc = (int)cooperative_groups::this_cluster().num_blocks();
  const int rank = (int)cooperative_groups::this_cluster().block_rank();
  const int64_t g = blockIdx.x / kc;
  const Slice ps(q.np, rank, kc);
  const float* xg = x + g * q.n;
  const float* dpg = dp + g * q.np;
  const uint8_t* cg = code + g * q.np;
  const float* gg = gdx ? gdx + g * q.n : nullptr;
  const float m = mean[g], r = rstd[g], ga = gamma[g];
  const float gdg = gdgamma ? gdgamma[g] : 0.f, gdb = gdbeta ? gdbeta[g] : 0.f;
  const double nd = (double)q.n;
  // sums: G1 = sum gdx, Gx = sum gdx*xh, Gd = sum gdx*dy (windows, then leftovers)
  const Slice ls(q.nl, rank, kc);
  double v[3] = {0.0, 0.0, 0.0};
  if (gg) {
    for (int p = ps.lo + threadIdx.x; p < ps.hi; p += blockDim.x) {
      const int e0 = q.elem0(p);
      const uint8_t c = cg[p];
      const float dl = dpg[p];  // unconditional: no code -> load dependence
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int e = e0 + q.off(k);
        const float t = gg[e];
        v[0] += (double)t;
        v[1] += (double)t * (double)((xg[e] - m) * r);
        if (c == k) v[2] += (double)dl * (double)t;
      }
    }
    for (int j = ls.lo + threadIdx.x; j < ls.hi; j += blockDim.x) {
      const int e = q.left(j);
      const float t = gg[e];
      v[0] += (double)t;
      v[1] += (double)t * (double)((xg[e] - m) * r);
    }
  }
  cluster_sum<3>(v, sm, part);
  const double A = (double)dbeta[g] / nd, Bm = (double)dgamma[g] / nd;
  const double G1 = v[0], Gx = v[1], GD = v[2] - A * G1;
  const double gr = (double)ga * (double)r;
  if (threadIdx.x == 0 && rank == 0) g_gamma[g] = (float)((double)r * (GD - Bm * Gx));
  // h = -gr*(dy*Gx/n + Bm*gdx) + gdg*dy = dy*ch + gdx*cgd
  const double mean_h = -gr * (A * Gx + Bm * G1) / nd + gdg * A;
  const double mean_hx = -2.0 * gr * Bm * Gx / nd + gdg * Bm;
  const double kx = gr * (double)r * (GD - Bm * Gx) / nd;
  const float ch = (float)(-gr * Gx / nd + gdg), cgd = (float)(-gr * Bm);
  const float mh = (float)mean_h, mhx = (float)mean_hx, fkx = (float)kx;
  // g_x over the windows (with g_dy at the routed position -> g_dp), then leftovers;
  // g_dy = gr*(gdx - G1/n - xh*Gx/n) + gdg*xh + gdb
  const float fgr = (float)gr, g1n = (float)(G1 / nd), gxn = (float)(Gx / nd);
  float* gxg = g_x + g * q.n;
  float* gdpg = g_dp + g * q.np;
  for (int p = ps.lo + threadIdx.x; p < ps.hi; p += blockDim.x) {
    const int e0 = q.elem0(p);
    const uint8_t c = cg[p];
    const float dl = dpg[p], d = c != kOff ? dl : 0.f;  // unconditional load
    float o = 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = e0 + q.off(k);
      const float xh = (xg[e] - m) * r;
      const float t = gg ? gg[e] : 0.f;
      const float dy = c == k ? d : 0.f;
      gxg[e] = r * ((dy * ch + t * cgd) - mh - xh * mhx) - fkx * xh;
      if (c == k) o = fgr * (t - g1n - xh * gxn) + gdg * xh + gdb;
    }
    gdpg[p] = o;
  }
  for (int j = ls.lo + threadIdx.x; j < ls.hi; j += blockDim.x) {
    const int e = q.left(j);
    const float xh = (xg[e] - m) * r;
    const float t = gg ? gg[e] : 0.f;
    gxg[e] = r * (t * cgd - mh - xh * mhx) - fkx * xh;
  }
}

// ------------------------------------------- smem-resident forward
// The CTA's slice of the group (a contiguous range of images, so every
// window of those images is inside it) is bulk-copied from HBM ONCE into
// shared memory by the TMA engine (cp.async.bulk + mbarrier); the statistics
// pass and the window pass both read the copy. The 2-pass kernel above
// re-reads the group, and at 32 tasks the groups in flight exceed L2
// (measured: 572 vs 844 us per outer step's forward launches, ncu). The same
// staging for the two backward kernels measured no faster (their window
// passes, which write the full-size dx, dominate), so they stay 2-pass.

// One-shot bulk (TMA engine) copy of `nbytes` from global into shared memory,
// completion tracked by a shared mbarrier; every thread of the CTA returns
// after the data has landed. src/dst 16-byte aligned, nbytes % 16 == 0.
__device__ __forceinline__ void bulk_load2(void* dst0, const void* src0, uint32_t b0, void* dst1,
                                           const void* src1, uint32_t b1, uint64_t* bar) {
  const uint32_t sbar = (uint32_t)__cvta_generic_to_shared(bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"(b0 + b1)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(dst0)),
        "l"(src0), "r"(b0), "r"(sbar)
        : "memory");
    if (b1)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              (uint32_t)__cvta_generic_to_shared(dst1)),
          "l"(src1), "r"(b1), "r"(sbar)
          : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAITB_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
      "@!p bra WAITB_%=;\n\t}" ::"r"(sbar)
      : "memory");
}

struct ImgSlice {
  int b0, b1;  // images [b0, b1)
  __device__ ImgSlice(int B, int r, int k) {
    b0 = (int)((int64_t)B * r / k);
    b1 = (int)((int64_t)B * (r + 1) / k);
  }
};

__global__ void bnpool_fwd_smem(int B, int H, int W, const float* __restrict__ x,
                                const float* __restrict__ gamma, const float* __restrict__ beta,
                                double eps, float* __restrict__ out, uint8_t* __restrict__ code,
                                float* __restrict__ mean_out, float* __restrict__ rstd_out,
                                float* __restrict__ cols) {
  extern __shared__ float xs[];
  __shared__ double sm[32 * 2 + 2];
  __shared__ double part[2];
  const Geo q(B, H, W);
  const int kc = (int)cooperative_groups::this_cluster().num_blocks();
  const int rank = (int)cooperative_groups::this_cluster().block_rank();
  const int64_t g = blockIdx.x / kc;
  const ImgSlice is(B, rank, kc);
  const int e0 = is.b0 * q.HW, ne = (is.b1 - is.b0) * q.HW;
  const float* xg = x + g * q.n + e0;
  __shared__ uint64_t bar;
  bulk_load2(xs, xg, (uint32_t)ne * 4, nullptr, nullptr, 0, &bar);
  double v[2] = {0.0, 0.0};
  for (int i = threadIdx.x; i < ne; i += blockDim.x) {
    const float a = xs[i];
    v[0] += (double)a;
    v[1] += (double)a * (double)a;
  }
  cluster_sum<2>(v, sm, part);
  const double mu = v[0] / q.n;
  double var = v[1] / q.n - mu * mu;
  var = var > 0.0 ? var : 0.0;
  const double rd = 1.0 / sqrt(var + eps);
  const float m = (float)mu, r = (float)rd, ga = gamma[g], be = beta[g];
  if (threadIdx.x == 0 && rank == 0) {
    mean_out[g] = m;
    rstd_out[g] = r;
  }
  const float s = ga * r;
  float* og = out + g * q.np;
  uint8_t* cg = code + g * q.np;
  float* c9 = cols ? cols + g * 9 * (int64_t)q.np : nullptr;
  for (int p = is.b0 * q.P2 + threadIdx.x; p < is.b1 * q.P2; p += blockDim.x) {
    const int e = q.elem0(p) - e0;
    const float x0 = xs[e], x1 = xs[e + 1], x2 = xs[e + W], x3 = xs[e + W + 1];
    float best = s * (x0 - m) + be;
    int kb = 0;
    float z1 = s * (x1 - m) + be;
    if (z1 > best) best = z1, kb = 1;
    float z2 = s * (x2 - m) + be;
    if (z2 > best) best = z2, kb = 2;
    float z3 = s * (x3 - m) + be;
    if (z3 > best) best = z3, kb = 3;
    const bool on = best > 0.f;
    og[p] = on ? best : 0.f;
    cg[p] = on ? (uint8_t)kb : kOff;
    if (c9) q.scatter_cols(c9, p, on ? best : 0.f);
  }
}


// ------------------------------------------------ split-K NT GEMM (weight grads)
// C[t] (M x P) = A[t] (M x N) . B[t]^T (P x N): both operands contiguous along
// the contraction axis n, which is long (B*H*W, up to 58,800) while M x P is
// small (64 x 576): the convolution weight-gradient shape. cuBLAS runs it
// with one CTA per 32x32 output tile walking all of n (36 CTAs per task), so
// at a few tasks per GPU most SMs idle. Here n is split into S ranges, each
// CTA computes a 64x64 tile over its range in fp32 (SIMT FFMA: the path must
// keep fp32 accuracy, reading Z16 / DESIGN §8), and a second kernel sums the
// S partials in fixed order (bitwise reproducible).
constexpr int GM = 64, GK = 32, GTHREADS = 128, GTM = 8, GPAD = 4;

// CTA tile GM x GP (GP = 16*TP) over one n-range; 128 threads as 16 (p) x 8 (m),
// each an 8 x TP register tile. Operands are staged k-major in shared memory:
// every thread loads 4 consecutive rows at one n (coalesced along n across
// the warp) and stores them as one 16-byte vector, so stores are
// conflict-free and the inner loop reads 16-byte vectors.
template <int TP>
__global__ void __launch_bounds__(GTHREADS) gemm_nt_partial(int M, int P, int N, int ptiles,
                                                            int cps, const float* __restrict__ A,
                                                            const float* __restrict__ B,
                                                            float* __restrict__ out,
                                                            int64_t out_t_stride,
                                                            int64_t out_s_stride, int S1,
                                                            const float* __restrict__ A2,
                                                            const float* __restrict__ B2) {
  constexpr int GP = 16 * TP;
  constexpr int AG = GM / 16, BG = GP / 16;  // 4-row groups per warp
  __shared__ __align__(16) float As[2][GK][GM + GPAD];
  __shared__ __align__(16) float Bs[2][GK][GP + GPAD];
  // splits [0, S1) contract (A, B), splits [S1, 2 S1) the second pair (A2, B2)
  const int t = blockIdx.z, s = blockIdx.y, second = s >= S1, sl = second ? s - S1 : s;
  const int mt = blockIdx.x / ptiles, pt = blockIdx.x - mt * ptiles;
  const int m0 = mt * GM, p0 = pt * GP;
  const int nch = (N + GK - 1) / GK;
  const int c0 = sl * cps, c1 = min(nch, c0 + cps);
  const float* At = (second ? A2 : A) + (int64_t)t * M * N;
  const float* Bt = (second ? B2 : B) + (int64_t)t * P * N;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // p: tx*TP.., m: ty*8..
  float4 ra[AG], rb[BG];
  auto row = [&](const float* base, int r, int lim, int n, bool nok) {
    return (nok && r < lim) ? __ldg(base + (int64_t)r * N + n) : 0.f;
  };
  auto load = [&](int c) {
    const int n = c * GK + lane;
    const bool nok = n < N;
#pragma unroll
    for (int j = 0; j < AG; ++j) {
      const int r = m0 + warp * (GM / 4) + 4 * j;
      ra[j] = make_float4(row(At, r, M, n, nok), row(At, r + 1, M, n, nok),
                          row(At, r + 2, M, n, nok), row(At, r + 3, M, n, nok));
    }
#pragma unroll
    for (int j = 0; j < BG; ++j) {
      const int r = p0 + warp * (GP / 4) + 4 * j;
      rb[j] = make_float4(row(Bt, r, P, n, nok), row(Bt, r + 1, P, n, nok),
                          row(Bt, r + 2, P, n, nok), row(Bt, r + 3, P, n, nok));
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int j = 0; j < AG; ++j)
      *reinterpret_cast<float4*>(&As[buf][lane][warp * (GM / 4) + 4 * j]) = ra[j];
#pragma unroll
    for (int j = 0; j < BG; ++j)
      *reinterpret_cast<float4*>(&Bs[buf][lane][warp * (GP / 4) + 4 * j]) = rb[j];
  };
  float acc[GTM][TP];
#pragma unroll
  for (int i = 0; i < GTM; ++i)
#pragma unroll
    for (int j = 0; j < TP; ++j) acc[i][j] = 0.f;
  if (c0 < c1) {
    load(c0);
    store(0);
    __syncthreads();
    for (int c = c0; c < c1; ++c) {
      const int buf = (c - c0) & 1;
      if (c + 1 < c1) load(c + 1);
#pragma unroll 8
      for (int k = 0; k < GK; ++k) {
        const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][k][ty * GTM]);
        const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][k][ty * GTM + 4]);
        const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        float bv[TP];
        if constexpr (TP == 4) {
          const float4 b = *reinterpret_cast<const float4*>(&Bs[buf][k][tx * 4]);
          bv[0] = b.x, bv[1] = b.y, bv[2] = b.z, bv[3] = b.w;
        } else {
#pragma unroll
          for (int j = 0; j < TP; ++j) bv[j] = Bs[buf][k][tx * TP + j];
        }
#pragma unroll
        for (int i = 0; i < GTM; ++i)
#pragma unroll
          for (int j = 0; j < TP; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      if (c + 1 < c1) store(buf ^ 1);
      __syncthreads();
    }
  }
  float* o = out + (int64_t)t * out_t_stride + (int64_t)s * out_s_stride;
#pragma unroll
  for (int i = 0; i < GTM; ++i) {
    const int m = m0 + ty * GTM + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < TP; ++j) {
      const int p = p0 + tx * TP + j;
      if (p < P) o[(int64_t)m * P + p] = acc[i][j];
    }
  }
}

// C[t][e] (+)= sum over s (in order) of part[t][s][e], e < M*P
__global__ void gemm_nt_reduce(int64_t MP, int S, const float* __restrict__ part,
                               float* __restrict__ C, int accumulate) {
  const int64_t t = blockIdx.y;
  const float* pt = part + t * S * MP;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < MP;
       e += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < S; ++s) acc += pt[(int64_t)s * MP + e];
    C[t * MP + e] = accumulate ? C[t * MP + e] + acc : acc;
  }
}

struct SplitPlan {
  int tp, ptiles, mtiles, S, cps;
};

int resident_slots(int tp) {  // CTAs of gemm_nt_partial<tp> resident on the device
  static int cached[5] = {0, 0, 0, 0, 0};
  if (!cached[tp]) {
    int dev = 0, sms = 148, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (tp == 4)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gemm_nt_partial<4>, GTHREADS, 0);
    else
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gemm_nt_partial<1>, GTHREADS, 0);
    cached[tp] = (occ > 0 ? occ : 1) * (sms > 0 ? sms : 148);
  }
  return cached[tp];
}

SplitPlan split_plan(int64_t T, int64_t M, int64_t P, int64_t N, int64_t min_chunks = 8) {
  SplitPlan q;
  q.tp = P <= 16 ? 1 : 4;
  const int GP = 16 * q.tp;
  q.mtiles = (int)((M + GM - 1) / GM);
  q.ptiles = (int)((P + GP - 1) / GP);
  const int64_t nch = (N + GK - 1) / GK;
  const int64_t tiles = T * q.mtiles * q.ptiles;
  const int64_t slots = resident_slots(q.tp);
  int64_t most = nch / min_chunks;  // each split walks >= min_chunks chunks (default 256 of n)
  if (most < 1) most = 1;
  if (most > 4096) most = 4096;
  // fewest splits whose CTA count fills the resident slots' waves to >= 90%
  // (first wave full); with few tiles, as many as `most` allows
  int64_t S = 1;
  double best = -1.0;
  for (int64_t c = 1; c <= most; ++c) {
    const int64_t ctas = tiles * c;
    const int64_t waves = (ctas + slots - 1) / slots;
    const double fill = (double)ctas / (double)(waves * slots);
    const double score = waves == 1 ? fill : fill + 0.001 * (double)waves;
    if (score > best + 1e-9) {
      best = score;
      S = c;
    }
    if (waves == 1 && fill >= 0.9) break;
    if (waves > 1 && fill >= 0.9) break;
  }
  q.cps = (int)((nch + S - 1) / S);
  q.S = (int)((nch + q.cps - 1) / q.cps);
  if (q.S < 1) q.S = 1;
  return q;
}

bool geo_ok(int64_t G, int64_t B, int64_t H, int64_t W, bool pool) {
  if (G < 0 || B < 1 || H < 1 || W < 1) return false;
  if (pool && (H < 2 || W < 2)) return false;
  if (B * H * W > (int64_t)1 << 30) return false;
  return G < ((int64_t)1 << 31) / 9;
}

dim3 stream_grid(int64_t rows, int64_t n) {
  // enough blocks to fill 148 SMs x 8 resident blocks; each loops inside its row
  int64_t chunks = (148 * 8 + rows - 1) / rows, most = (n + 255) / 256;
  if (chunks > most) chunks = most;
  if (chunks > 65535) chunks = 65535;
  if (chunks < 1) chunks = 1;
  return dim3((unsigned)rows, (unsigned)chunks);
}

constexpr int kBnThreads = 256;
constexpr int kSmemCap = 64 * 1024;  // per-CTA slice budget (>= 3 CTAs per SM)

// CTAs per group (cluster size): enough groups-x-slices to give every SM
// ~8 CTAs, each slice >= 4096 elements; portable cluster sizes 1, 2, 4, 8.
// Also split groups larger than kSliceCap elements (the 28x28 layer's
// 19,600 at 25 images) so 32-task grids end in a finer last wave: 2 CTAs
// per group measured 128 vs 137 us (backward), 172 vs 182 us (second
// derivative); smaller slices lose more to the cluster reduction
// (profiles/r01f_bn_slice_sweep.txt). NET_BN_SLICE overrides (0 = off).
constexpr int64_t kSliceCap = 16384;
int cluster_for(int64_t G, int64_t n) {
  static const int64_t slice_cap = [] {
    const char* e = getenv("NET_BN_SLICE");
    return e ? (int64_t)atoll(e) : kSliceCap;
  }();
  // smallest per-CTA slice when splitting only to fill the GPU: below ~4K
  // elements the cluster reduction and per-CTA fixed costs outweigh the
  // extra CTAs (measured, explicit MAML step at 4 tasks: 1024 -> 5.46 ms,
  // 2048 -> 5.32, 4096 -> 5.23, no fill splitting -> 5.28; 32 tasks, whose
  // splits come from the slice cap, unchanged: profiles/r02x_bn_min_slice.txt).
  // With concurrent task chains and the cuBLAS SM hint, 8192 is as fast at
  // 4 tasks and faster at 8 (8.09 -> 7.97 ms) and 16 (14.75 -> 14.70):
  // profiles/r02bn_bn_min_slice_8k.txt
  static const int64_t min_slice = [] {
    const char* e = getenv("NET_BN_MIN_SLICE");
    return e ? (int64_t)atoll(e) : (int64_t)8192;
  }();
  const int64_t want = 148 * 8;
  int kc = 1;
  while (kc < 8 && ((G * kc < want && n / (2 * kc) >= min_slice) ||
                    (slice_cap > 0 && n / kc > slice_cap)))
    kc *= 2;
  return kc;
}

// smem-resident plan (bulk-copied slices): the smallest cluster (>= cluster_for) whose image slice
// of `arrays` fp32 arrays fits kSmemCap; 0 if none does
int smem_cluster(int64_t G, int64_t B, int64_t HW, int arrays, size_t* bytes) {
  if (HW % 4 != 0) return 0;  // bulk copies need 16-byte aligned image slices
  for (int kc = cluster_for(G, B * HW); kc <= 8; kc *= 2) {
    if (kc > B) break;
    const int64_t imgs = (B + kc - 1) / kc;
    const size_t need = (size_t)imgs * HW * 4 * arrays;
    if (need <= (size_t)kSmemCap) {
      *bytes = need;
      return kc;
    }
  }
  return 0;
}

template <typename... KArgs, typename... Args>
int launch_clustered(void (*kernel)(KArgs...), int64_t G, int kc, size_t smem, cudaStream_t st,
                     Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(G * kc));
  cfg.blockDim = dim3(kBnThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)kc;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemCap) !=
          cudaSuccess) {
    g_err = "cannot raise the dynamic shared-memory limit";
    return NET_ECUDA;
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, args...);
  if (e != cudaSuccess) {
    g_err = cudaGetErrorString(e);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return NET_ECUDA;
  }
  return launched();
}

template <typename... KArgs, typename... Args>
int launch_group_kernel(void (*kernel)(KArgs...), int64_t G, int64_t n, cudaStream_t st,
                        Args... args) {
  return launch_clustered(kernel, G, cluster_for(G, n), 0, st, args...);
}

// ------------------------------------------- forward-mode (JVP) kernels
// The hand-scheduled second-order MAML step (maml.ExplicitMaml) gets the
// Hessian-vector products of the inner loss by forward-over-reverse
// differentiation: tangents (ẋ, γ̇, β̇) ride along the forward pass and the
// backward pass. Formulas: include/mamlnet.h (net_bnpool_jvp,
// net_bnpool_bwd_jvp); derivation DESIGN.md §8.2.

// JVP of bnpool_fwd at (x, gamma, beta) along (xd, gd, bd): one CTA cluster
// per group; pass 1 the group sums S1 = sum xd, S2 = sum xh*xd (fp64),
// pass 2 the pooled tangent at each active window's maximum.
__global__ void __launch_bounds__(256, 6) bnpool_jvp_kernel(
    int B, int H, int W, const float* __restrict__ x, const float* __restrict__ xd,
    const float* __restrict__ gamma, const float* __restrict__ gd, const float* __restrict__ bd,
    const uint8_t* __restrict__ code, const float* __restrict__ mean,
    const float* __restrict__ rstd, float* __restrict__ outd, float* __restrict__ s1,
    float* __restrict__ s2, float* __restrict__ cols) {
  __shared__ double sm[32 * 2 + 2];
  __shared__ double part[2];
  const Geo q(B, H, W);
  const int kc = (int)cooperative_groups::this_cluster().num_blocks();
  const int rank = (int)cooperative_groups::this_cluster().block_rank();
  const int64_t g = blockIdx.x / kc;
  const Slice es(q.n, rank, kc), ps(q.np, rank, kc);
  const float* xg = x + g * q.n;
  const float* xdg = xd + g * q.n;
  const float m = mean[g], r = rstd[g];
  double v[2] = {0.0, 0.0};
  // 16-byte loads over the 4-aligned middle of the slice, scalar ends
  const bool al = (((uintptr_t)xg | (uintptr_t)xdg) & 15) == 0;
  int va = al ? min((es.lo + 3) & ~3, es.hi) : es.hi, vb = al ? max(es.hi & ~3, va) : es.hi;
  for (int i4 = (va >> 2) + threadIdx.x; i4 < (vb >> 2); i4 += blockDim.x) {
    const float4 t = reinterpret_cast<const float4*>(xdg)[i4];
    const float4 x4 = reinterpret_cast<const float4*>(xg)[i4];
    v[0] += (double)t.x + (double)t.y + (double)t.z + (double)t.w;
    v[1] += (double)t.x * (double)((x4.x - m) * r) + (double)t.y * (double)((x4.y - m) * r) +
            (double)t.z * (double)((x4.z - m) * r) + (double)t.w * (double)((x4.w - m) * r);
  }
  for (int i = es.lo + threadIdx.x; i < va; i += blockDim.x) {
    const float t = xdg[i];
    v[0] += (double)t;
    v[1] += (double)t * (double)((xg[i] - m) * r);
  }
  for (int i = vb + threadIdx.x; i < es.hi; i += blockDim.x) {
    const float t = xdg[i];
    v[0] += (double)t;
    v[1] += (double)t * (double)((xg[i] - m) * r);
  }
  cluster_sum<2>(v, sm, part);
  const float a = (float)(v[0] / q.n), b = (float)(v[1] / q.n);
  if (threadIdx.x == 0 && rank == 0) {
    s1[g] = a;
    s2[g] = b;
  }
  const float ga = gamma[g], gdd = gd ? gd[g] : 0.f, bdd = bd ? bd[g] : 0.f;
  const uint8_t* cg = code + g * q.np;
  float* og = outd + g * q.np;
  float* c9 = cols ? cols + g * 9 * (int64_t)q.np : nullptr;
  for (int p = ps.lo + threadIdx.x; p < ps.hi; p += blockDim.x) {
    const uint8_t c = cg[p];
    float o = 0.f;
    if (c != kOff) {
      const int e = q.elem0(p) + q.off(c);
      const float xh = (xg[e] - m) * r;
      const float xhd = r * (xdg[e] - a - xh * b);
      o = gdd * xh + ga * xhd + bdd;
    }
    og[p] = o;
    if (c9) q.scatter_cols(c9, p, o);
  }
}

// JVP of bnpool_bwd at (dp, x, gamma) along (dpd, xd, gd), with S1/n, S2/n
// from bnpool_jvp of the same xd. Pass 1 (pooled): P1 = sum dyd,
// P2 = sum dyd*xh, P3 = sum dy*xhd; pass 2 (every element) the tangent of dx.
// dgd/dbd are ACCUMULATED (+=).
template <int MINB, bool EVEN>  // EVEN: W even, window rows as float2 pairs
__global__ void __launch_bounds__(256, MINB) bnpool_bwd_jvp_kernel(
    int B, int H, int W, const float* __restrict__ dp, const float* __restrict__ dpd,
    const uint8_t* __restrict__ code, const float* __restrict__ x, const float* __restrict__ xd,
    const float* __restrict__ gamma, const float* __restrict__ gd, const float* __restrict__ mean,
    const float* __restrict__ rstd, const float* __restrict__ dgamma,
    const float* __restrict__ dbeta, const float* __restrict__ s1, const float* __restrict__ s2,
    float* __restrict__ dxd, float* __restrict__ dgd_acc, float* __restrict__ dbd_acc) {
  __shared__ double sm[32 * 3 + 3];
  __shared__ double part[3];
  const Geo q(B, H, W);
  const int kc = (int)cooperative_groups::this_cluster().num_blocks();
  const int rank = (int)cooperative_groups::this_cluster().block_rank();
  const int64_t g = blockIdx.x / kc;
  const Slice ps(q.np, rank, kc);
  const float* xg = x + g * q.n;
  const float* xdg = xd + g * q.n;
  const float* dpg = dp + g * q.np;
  const float* dpdg = dpd + g * q.np;
  const uint8_t* cg = code + g * q.np;
  const float m = mean[g], r = rstd[g], a = s1[g], b = s2[g];
  double v[3] = {0.0, 0.0, 0.0};
  for (int p = ps.lo + threadIdx.x; p < ps.hi; p += blockDim.x) {
    const uint8_t c = cg[p];
    const float d = dpg[p], dd = dpdg[p];  // unconditional: only the x gathers depend on the code
    if (c != kOff) {
      const int e = q.elem0(p) + q.off(c);
      const float xh = (xg[e] - m) * r;
      const float xhd = r * (xdg[e] - a - xh * b);
      v[0] += (double)dd;
      v[1] += (double)dd * (double)xh;
      v[2] += (double)d * (double)xhd;
    }
  }
  cluster_sum<3>(v, sm, part);
  const double nd = (double)q.n;
  if (threadIdx.x == 0 && rank == 0) {
    if (dbd_acc) dbd_acc[g] += (float)v[0];
    if (dgd_acc) dgd_acc[g] += (float)(v[1] + v[2]);
  }
  const float ga = gamma[g], gdd = gd ? gd[g] : 0.f;
  const float A = (float)((double)dbeta[g] / nd), Bm = (float)((double)dgamma[g] / nd);
  const float Ad = (float)(v[0] / nd), Bmd = (float)((v[1] + v[2]) / nd);
  // dxd = c1*D + c2*Dd, D = dy - A - xh*Bm, Dd = dyd - Ad - xhd*Bm - xh*Bmd
  const float c1 = gdd * r - ga * r * r * b, c2 = ga * r;
  float* og = dxd + g * q.n;
  for (int p = ps.lo + threadIdx.x; p < ps.hi; p += blockDim.x) {
    const int e0 = q.elem0(p);
    const uint8_t c = cg[p];
    const float dl = dpg[p], ddl = dpdg[p];
    const float d = c != kOff ? dl : 0.f, dd = c != kOff ? ddl : 0.f;
    if constexpr (EVEN) {
      const float2 t0 = *reinterpret_cast<const float2*>(xg + e0);
      const float2 t1 = *reinterpret_cast<const float2*>(xg + e0 + W);
      const float2 u0 = *reinterpret_cast<const float2*>(xdg + e0);
      const float2 u1 = *reinterpret_cast<const float2*>(xdg + e0 + W);
      const float xv[4] = {t0.x, t0.y, t1.x, t1.y}, xdv[4] = {u0.x, u0.y, u1.x, u1.y};
      float o[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float xh = (xv[k] - m) * r;
        const float xhd = r * (xdv[k] - a - xh * b);
        const float D = (c == k ? d : 0.f) - A - xh * Bm;
        const float Dd = (c == k ? dd : 0.f) - Ad - xhd * Bm - xh * Bmd;
        o[k] = c1 * D + c2 * Dd;
      }
      *reinterpret_cast<float2*>(og + e0) = make_float2(o[0], o[1]);
      *reinterpret_cast<float2*>(og + e0 + W) = make_float2(o[2], o[3]);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int e = e0 + q.off(k);
        const float xh = (xg[e] - m) * r;
        const float xhd = r * (xdg[e] - a - xh * b);
        const float D = (c == k ? d : 0.f) - A - xh * Bm;
        const float Dd = (c == k ? dd : 0.f) - Ad - xhd * Bm - xh * Bmd;
        og[e] = c1 * D + c2 * Dd;
      }
    }
  }
  const Slice ls(q.nl, rank, kc);
  for (int j = ls.lo + threadIdx.x; j < ls.hi; j += blockDim.x) {
    const int e = q.left(j);
    const float xh = (xg[e] - m) * r;
    const float xhd = r * (xdg[e] - a - xh * b);
    og[e] = c1 * (-A - xh * Bm) + c2 * (-Ad - xhd * Bm - xh * Bmd);
  }
}

// ------------------------------------------- classifier head (fc + cross entropy)
// One CTA per task: feat[b][c] = h4[t][c][b] (the 1x1 pooled map), logits =
// feat.Wfc^T + bfc, per-task mean cross entropy over its B images, and the
// whole backward of that loss. Shared memory: feat [C][B] (+ tangent),
// W [J][C] (+ tangent), probabilities and dlogits [B][J].
constexpr int kHeadThreads = 256;

// smem[0..count) = src[0..count) with 16-byte loads when both are aligned
// (all loads issued before the stores: one latency, not one per element).
__device__ __forceinline__ void stage(float* __restrict__ dst, const float* __restrict__ src,
                                      int count) {
  if ((((uintptr_t)src | (uintptr_t)dst) & 15) == 0) {
    const int c4 = count >> 2;
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* d4 = reinterpret_cast<float4*>(dst);
    int i = threadIdx.x;
    for (; i + 3 * (int)blockDim.x < c4; i += 4 * blockDim.x) {
      const float4 a = __ldg(s4 + i), b = __ldg(s4 + i + blockDim.x),
                   c = __ldg(s4 + i + 2 * blockDim.x), d = __ldg(s4 + i + 3 * blockDim.x);
      d4[i] = a, d4[i + blockDim.x] = b, d4[i + 2 * blockDim.x] = c, d4[i + 3 * blockDim.x] = d;
    }
    for (; i < c4; i += blockDim.x) d4[i] = __ldg(s4 + i);
    for (int j = (c4 << 2) + threadIdx.x; j < count; j += blockDim.x) dst[j] = __ldg(src + j);
  } else {
#pragma unroll 4
    for (int j = threadIdx.x; j < count; j += blockDim.x) dst[j] = __ldg(src + j);
  }
}

__device__ __forceinline__ float block_sum_f(float v, float* red) {
  // fixed-order block sum (warp xor tree, then warp totals in order)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float s = 0.f;
  for (int w = 0; w < nw; ++w) s += red[w];
  return s;
}

__global__ void __launch_bounds__(kHeadThreads) fc_xent_kernel(
    int B, int C, int J, float inv_b, const float* __restrict__ h4, const float* __restrict__ Wfc,
    const float* __restrict__ bfc, const int64_t* __restrict__ labels, float* __restrict__ loss,
    float* __restrict__ prob, float* __restrict__ dW, float* __restrict__ db,
    float* __restrict__ dh4) {
  extern __shared__ float hs[];
  float* f = hs;              // [C][B]
  float* w = f + C * B;       // [J][C]
  float* pr = w + J * C;      // [B][J] probabilities, then dlogits
  __shared__ float red[32];
  const int64_t t = blockIdx.x;
  const float* ht = h4 + t * C * B;
  stage(f, ht, C * B);
  stage(w, Wfc + t * J * C, J * C);
  __syncthreads();
  for (int o = threadIdx.x; o < B * J; o += blockDim.x) {
    const int b = o / J, j = o - b * J;
    float z = bfc[t * J + j];
    for (int c = 0; c < C; ++c) z = fmaf(f[c * B + b], w[j * C + c], z);
    pr[o] = z;
  }
  __syncthreads();
  float lsum = 0.f;
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    float* z = pr + b * J;
    float mx = z[0];
    for (int j = 1; j < J; ++j) mx = fmaxf(mx, z[j]);
    float se = 0.f;
    for (int j = 0; j < J; ++j) se += expf(z[j] - mx);
    const int y = (int)labels[t * B + b];
    lsum += logf(se) + mx - z[y];
    const float ise = 1.f / se;
    for (int j = 0; j < J; ++j) {
      const float p = expf(z[j] - mx) * ise;
      prob[(t * B + b) * J + j] = p;
      z[j] = (p - (j == y ? 1.f : 0.f)) * inv_b;  // dlogits
    }
  }
  lsum = block_sum_f(lsum, red);
  if (threadIdx.x == 0) loss[t] = lsum * inv_b;
  __syncthreads();
  for (int o = threadIdx.x; o < J * C; o += blockDim.x) {
    const int j = o / C, c = o - j * C;
    float s = 0.f;
    for (int b = 0; b < B; ++b) s = fmaf(pr[b * J + j], f[c * B + b], s);
    dW[t * J * C + o] = s;
  }
  for (int j = threadIdx.x; j < J; j += blockDim.x) {
    float s = 0.f;
    for (int b = 0; b < B; ++b) s += pr[b * J + j];
    db[t * J + j] = s;
  }
  for (int o = threadIdx.x; o < C * B; o += blockDim.x) {
    const int c = o / B, b = o - c * B;
    float s = 0.f;
    for (int j = 0; j < J; ++j) s = fmaf(pr[b * J + j], w[j * C + c], s);
    dh4[t * C * B + o] = s;
  }
}

// JVP of fc_xent's gradient outputs along (h4d, Wd, bd); dWd/dbd accumulated.
__global__ void __launch_bounds__(kHeadThreads) fc_xent_jvp_kernel(
    int B, int C, int J, float inv_b, const float* __restrict__ h4, const float* __restrict__ h4d,
    const float* __restrict__ Wfc, const float* __restrict__ Wd, const float* __restrict__ bd,
    const int64_t* __restrict__ labels, const float* __restrict__ prob,
    float* __restrict__ dWd_acc, float* __restrict__ dbd_acc, float* __restrict__ dh4d) {
  extern __shared__ float hs[];
  float* f = hs;              // [C][B]
  float* fd = f + C * B;      // [C][B]
  float* w = fd + C * B;      // [J][C]
  float* wd = w + J * C;      // [J][C]
  float* dl = wd + J * C;     // [B][J] dlogits
  float* dld = dl + B * J;    // [B][J] their tangent
  const int64_t t = blockIdx.x;
  stage(f, h4 + t * C * B, C * B);
  if (h4d)
    stage(fd, h4d + t * C * B, C * B);
  else
    for (int i = threadIdx.x; i < C * B; i += blockDim.x) fd[i] = 0.f;
  stage(w, Wfc + t * J * C, J * C);
  if (Wd)
    stage(wd, Wd + t * J * C, J * C);
  else
    for (int i = threadIdx.x; i < J * C; i += blockDim.x) wd[i] = 0.f;
  __syncthreads();
  for (int o = threadIdx.x; o < B * J; o += blockDim.x) {  // logit tangents
    const int b = o / J, j = o - b * J;
    float z = bd ? bd[t * J + j] : 0.f;
    for (int c = 0; c < C; ++c) z = fmaf(fd[c * B + b], w[j * C + c], fmaf(f[c * B + b], wd[j * C + c], z));
    dld[o] = z;
  }
  __syncthreads();
  for (int b = threadIdx.x; b < B; b += blockDim.x) {  // softmax Jacobian
    const float* p = prob + (t * B + b) * J;
    const int y = (int)labels[t * B + b];
    float sp = 0.f;
    for (int j = 0; j < J; ++j) sp = fmaf(p[j], dld[b * J + j], sp);
    for (int j = 0; j < J; ++j) {
      dld[b * J + j] = p[j] * (dld[b * J + j] - sp) * inv_b;
      dl[b * J + j] = (p[j] - (j == y ? 1.f : 0.f)) * inv_b;
    }
  }
  __syncthreads();
  for (int o = threadIdx.x; o < J * C; o += blockDim.x) {
    const int j = o / C, c = o - j * C;
    float s = 0.f;
    for (int b = 0; b < B; ++b)
      s = fmaf(dld[b * J + j], f[c * B + b], fmaf(dl[b * J + j], fd[c * B + b], s));
    if (dWd_acc) dWd_acc[t * J * C + o] += s;
  }
  for (int j = threadIdx.x; j < J; j += blockDim.x) {
    float s = 0.f;
    for (int b = 0; b < B; ++b) s += dld[b * J + j];
    if (dbd_acc) dbd_acc[t * J + j] += s;
  }
  for (int o = threadIdx.x; o < C * B; o += blockDim.x) {
    const int c = o / B, b = o - c * B;
    float s = 0.f;
    for (int j = 0; j < J; ++j)
      s = fmaf(dld[b * J + j], w[j * C + c], fmaf(dl[b * J + j], wd[j * C + c], s));
    dh4d[t * C * B + o] = s;
  }
}

// ------------------------------------------- sum over the task axis
// out[off[l] + i] = sum over t (in order) of in[T*off[l] + t*size_l + i]:
// the leaf-major [leaf][T][size] buffer of T tasks' parameter cotangents
// folded into one tree (theta_0 = phi broadcast -> its cotangent).
__global__ void task_sum_kernel(int64_t T, int64_t nl, const int64_t* __restrict__ off,
                                const float* __restrict__ in, float* __restrict__ out) {
  const int64_t n = off[nl];
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n;
       o += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = nl - 1;  // last leaf l with off[l] <= o
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (off[mid] <= o) lo = mid; else hi = mid - 1;
    }
    const int64_t size = off[lo + 1] - off[lo], i = o - off[lo];
    const float* src = in + T * off[lo] + i;
    float s = 0.f;
    for (int64_t t = 0; t < T; ++t) s += src[t * size];
    out[o] = s;
  }
}

}  // namespace

extern "C" {

int net_im2col3x3(int64_t G, int64_t B, int64_t H, int64_t W, const float* h, float* cols,
                  void* stream) {
  if (!geo_ok(G, B, H, W, false)) return fail("net_im2col3x3: bad geometry");
  if (G == 0) return NET_OK;
  if (!h || !cols) return fail("net_im2col3x3: NULL pointer");
  if ((B * H * W) % 4 == 0 && ((uintptr_t)cols & 15) == 0)  // float4 stores
    im2col4_kernel<<<stream_grid(G, B * H * W / 4), 256, 0, (cudaStream_t)stream>>>(
        (int)B, (int)H, (int)W, h, cols);
  else
    im2col_kernel<<<stream_grid(G, B * H * W), 256, 0, (cudaStream_t)stream>>>(
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

static int bnpool_fwd_run(const char* who, int64_t G, int64_t B, int64_t H, int64_t W,
                          const float* x, const float* gamma, const float* beta, double eps,
                          float* out, uint8_t* code, float* mean, float* rstd, float* cols,
                          void* stream) {
  if (!geo_ok(G, B, H, W, true)) return fail(std::string(who) + ": bad geometry");
  if (!(eps >= 0.0)) return fail(std::string(who) + ": eps must be >= 0");
  if (G == 0) return NET_OK;
  if (!x || !gamma || !beta || !out || !code || !mean || !rstd)
    return fail(std::string(who) + ": NULL pointer");
  size_t sb = 0;
  if (const int kc = ((uintptr_t)x & 15) ? 0 : smem_cluster(G, B, H * W, 1, &sb))
    return launch_clustered(bnpool_fwd_smem, G, kc, sb, (cudaStream_t)stream, (int)B, (int)H,
                            (int)W, x, gamma, beta, eps, out, code, mean, rstd, cols);
  return launch_group_kernel(bnpool_fwd_kernel, G, B * H * W, (cudaStream_t)stream, (int)B,
                             (int)H, (int)W, x, gamma, beta, eps, out, code, mean, rstd, cols);
}

int net_bnpool_fwd(int64_t G, int64_t B, int64_t H, int64_t W, const float* x,
                   const float* gamma, const float* beta, double eps, float* out, uint8_t* code,
                   float* mean, float* rstd, void* stream) {
  return bnpool_fwd_run("net_bnpool_fwd", G, B, H, W, x, gamma, beta, eps, out, code, mean, rstd,
                        nullptr, stream);
}

int net_bnpool_fwd_cols(int64_t G, int64_t B, int64_t H, int64_t W, const float* x,
                        const float* gamma, const float* beta, double eps, float* out,
                        uint8_t* code, float* mean, float* rstd, float* cols, void* stream) {
  if (!cols && G > 0) return fail("net_bnpool_fwd_cols: NULL cols");
  return bnpool_fwd_run("net_bnpool_fwd_cols", G, B, H, W, x, gamma, beta, eps, out, code, mean,
                        rstd, cols, stream);
}

int net_bnpool_bwd(int64_t G, int64_t B, int64_t H, int64_t W, const float* dp,
                   const uint8_t* code, const float* x, const float* gamma, const float* mean,
                   const float* rstd, float* dx, float* dgamma, float* dbeta, void* stream) {
  if (!geo_ok(G, B, H, W, true)) return fail("net_bnpool_bwd: bad geometry");
  if (G == 0) return NET_OK;
  if (!dp || !code || !x || !gamma || !mean || !rstd || !dx || !dgamma || !dbeta)
    return fail("net_bnpool_bwd: NULL pointer");
  const bool even = (W % 2 == 0) && ((uintptr_t)x & 7) == 0 && ((uintptr_t)dx & 7) == 0;
  return launch_group_kernel(even ? bnpool_bwd_kernel<true> : bnpool_bwd_kernel<false>, G,
                             B * H * W, (cudaStream_t)stream, (int)B, (int)H, (int)W, dp, code, x,
                             gamma, mean, rstd, dx, dgamma, dbeta);
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
  const int kc = cluster_for(G, B * H * W);
  const int64_t slice = B * H * W / kc;
  auto* kernel = slice > 2048 && slice <= 8192 ? bnpool_bwd2_kernel<8> : bnpool_bwd2_kernel<6>;
  return launch_clustered(kernel, G, kc, 0, (cudaStream_t)stream, (int)B, (int)H, (int)W, gdx,
                          gdgamma, gdbeta, dp, code, x, gamma, mean, rstd, dgamma, dbeta, g_dp, g_x,
                          g_gamma);
}

// C (+)= A.B^T (+ A2.B2^T): one partial launch over npairs x S n-ranges, then
// the fixed-order reduce (skipped only for one pair, S = 1, no accumulate).
static size_t gemm_nt_need(int64_t T, int64_t M, int64_t P, int64_t N, int npairs, int accumulate) {
  if (T <= 0 || M <= 0 || P <= 0 || N <= 0) return 0;
  SplitPlan q = split_plan(T * npairs, M, P, N);
  if (npairs == 1 && q.S == 1 && !accumulate) return 0;
  return (size_t)T * npairs * q.S * M * P * sizeof(float);
}

static int gemm_nt_run(const char* who, int64_t T, int64_t M, int64_t P, int64_t N,
                       const float* A, const float* B, const float* A2, const float* B2,
                       float* C, int accumulate, void* workspace, size_t workspace_bytes,
                       void* stream) {
  static thread_local std::string msg;
  auto bad = [&](const char* what) {
    msg = std::string(who) + ": " + what;
    return fail(msg.c_str());
  };
  if (T < 0 || M < 0 || P < 0 || N < 0 || T > 65535 || M > (1 << 20) || P > (1 << 20) ||
      N > ((int64_t)1 << 31) - 64 || M * N > ((int64_t)1 << 40))
    return bad("bad sizes");
  if (T == 0 || M == 0 || P == 0) return NET_OK;
  if (!C) return bad("NULL C");
  cudaStream_t st = (cudaStream_t)stream;
  if (N == 0) {
    if (accumulate) return NET_OK;
    if (cudaMemsetAsync(C, 0, (size_t)T * M * P * sizeof(float), st) != cudaSuccess)
      return bad("memset failed");
    return NET_OK;
  }
  if (!A || !B) return bad("NULL operand");
  if ((A2 == nullptr) != (B2 == nullptr)) return bad("A2 and B2 must both be given or both NULL");
  const int npairs = A2 ? 2 : 1;
  SplitPlan q = split_plan(T * npairs, M, P, N);
  const size_t need = gemm_nt_need(T, M, P, N, npairs, accumulate);
  if (need && (!workspace || workspace_bytes < need))
    return bad("workspace too small (see the *_workspace_bytes function)");
  const int slots = npairs * q.S;
  dim3 grid((unsigned)(q.mtiles * q.ptiles), (unsigned)slots, (unsigned)T);
  float* out = need ? (float*)workspace : C;
  const int64_t MP = M * P;
  if (q.tp == 4)
    gemm_nt_partial<4><<<grid, GTHREADS, 0, st>>>((int)M, (int)P, (int)N, q.ptiles, q.cps, A, B,
                                                   out, slots * MP, MP, q.S, A2, B2);
  else
    gemm_nt_partial<1><<<grid, GTHREADS, 0, st>>>((int)M, (int)P, (int)N, q.ptiles, q.cps, A, B,
                                                   out, slots * MP, MP, q.S, A2, B2);
  int rc = launched();
  if (rc != NET_OK || !need) return rc;
  int64_t blocks = (MP + 255) / 256;
  if (blocks > 1024) blocks = 1024;
  gemm_nt_reduce<<<dim3((unsigned)blocks, (unsigned)T), 256, 0, st>>>(MP, slots, out, C,
                                                                       accumulate);
  return launched();
}

size_t net_gemm_nt_workspace_bytes(int64_t T, int64_t M, int64_t P, int64_t N) {
  return gemm_nt_need(T, M, P, N, 1, 0);
}

int net_gemm_nt(int64_t T, int64_t M, int64_t P, int64_t N, const float* A, const float* B,
                float* C, void* workspace, size_t workspace_bytes, void* stream) {
  return gemm_nt_run("net_gemm_nt", T, M, P, N, A, B, nullptr, nullptr, C, 0, workspace,
                     workspace_bytes, stream);
}

size_t net_gemm_nt2_workspace_bytes(int64_t T, int64_t M, int64_t P, int64_t N, int npairs,
                                    int accumulate) {
  if (npairs != 1 && npairs != 2) return 0;
  return gemm_nt_need(T, M, P, N, npairs, accumulate != 0);
}

int net_gemm_nt2(int64_t T, int64_t M, int64_t P, int64_t N, const float* A, const float* B,
                 const float* A2, const float* B2, float* C, int accumulate, void* workspace,
                 size_t workspace_bytes, void* stream) {
  return gemm_nt_run("net_gemm_nt2", T, M, P, N, A, B, A2, B2, C, accumulate != 0, workspace,
                     workspace_bytes, stream);
}

static int bnpool_jvp_run(const char* who, int64_t G, int64_t B, int64_t H, int64_t W,
                          const float* x, const float* xd, const float* gamma, const float* gd,
                          const float* bd, const uint8_t* code, const float* mean,
                          const float* rstd, float* outd, float* s1, float* s2, float* cols,
                          void* stream) {
  if (!geo_ok(G, B, H, W, true)) return fail(std::string(who) + ": bad geometry");
  if (G == 0) return NET_OK;
  if (!x || !xd || !gamma || !code || !mean || !rstd || !outd || !s1 || !s2)
    return fail(std::string(who) + ": NULL pointer");
  return launch_group_kernel(bnpool_jvp_kernel, G, B * H * W, (cudaStream_t)stream, (int)B,
                             (int)H, (int)W, x, xd, gamma, gd, bd, code, mean, rstd, outd, s1, s2,
                             cols);
}

int net_bnpool_jvp(int64_t G, int64_t B, int64_t H, int64_t W, const float* x, const float* xd,
                   const float* gamma, const float* gd, const float* bd, const uint8_t* code,
                   const float* mean, const float* rstd, float* outd, float* s1, float* s2,
                   void* stream) {
  return bnpool_jvp_run("net_bnpool_jvp", G, B, H, W, x, xd, gamma, gd, bd, code, mean, rstd,
                        outd, s1, s2, nullptr, stream);
}

int net_bnpool_jvp_cols(int64_t G, int64_t B, int64_t H, int64_t W, const float* x,
                        const float* xd, const float* gamma, const float* gd, const float* bd,
                        const uint8_t* code, const float* mean, const float* rstd, float* outd,
                        float* s1, float* s2, float* cols, void* stream) {
  if (!cols && G > 0) return fail("net_bnpool_jvp_cols: NULL cols");
  return bnpool_jvp_run("net_bnpool_jvp_cols", G, B, H, W, x, xd, gamma, gd, bd, code, mean, rstd,
                        outd, s1, s2, cols, stream);
}

int net_bnpool_bwd_jvp(int64_t G, int64_t B, int64_t H, int64_t W, const float* dp,
                       const float* dpd, const uint8_t* code, const float* x, const float* xd,
                       const float* gamma, const float* gd, const float* mean, const float* rstd,
                       const float* dgamma, const float* dbeta, const float* s1, const float* s2,
                       float* dxd, float* dgd_acc, float* dbd_acc, void* stream) {
  if (!geo_ok(G, B, H, W, true)) return fail("net_bnpool_bwd_jvp: bad geometry");
  if (G == 0) return NET_OK;
  if (!dp || !dpd || !code || !x || !xd || !gamma || !mean || !rstd || !dgamma || !dbeta || !s1 ||
      !s2 || !dxd)
    return fail("net_bnpool_bwd_jvp: NULL pointer");
  const int kc = cluster_for(G, B * H * W);
  const int64_t slice = B * H * W / kc;
  (void)slice;  // <8> compiles spill-free (<6> spills 48 bytes): one variant for every slice
  const bool even = (W % 2 == 0) && (((uintptr_t)x | (uintptr_t)xd | (uintptr_t)dxd) & 7) == 0;
  return launch_clustered(even ? bnpool_bwd_jvp_kernel<8, true> : bnpool_bwd_jvp_kernel<8, false>,
                          G, kc, 0, (cudaStream_t)stream, (int)B, (int)H, (int)W, dp, dpd,
                          code, x, xd, gamma, gd, mean, rstd, dgamma, dbeta, s1, s2, dxd, dgd_acc,
                          dbd_acc);
}

static int head_smem(const void* kernel, size_t bytes) {
  if (bytes > 227 * 1024) return fail("head: B*C too large for shared memory");
  if (bytes > 48 * 1024 &&
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) !=
          cudaSuccess)
    return fail("head: cannot raise the dynamic shared-memory limit");
  return NET_OK;
}

int net_fc_xent(int64_t T, int64_t B, int64_t C, int64_t J, const float* h4, const float* Wfc,
                const float* bfc, const int64_t* labels, float* loss, float* prob, float* dW,
                float* db, float* dh4, void* stream) {
  if (T < 0 || B < 1 || C < 1 || J < 1 || T > 65535 || B * C > (1 << 24) || J > 1024)
    return fail("net_fc_xent: bad sizes");
  if (T == 0) return NET_OK;
  if (!h4 || !Wfc || !bfc || !labels || !loss || !prob || !dW || !db || !dh4)
    return fail("net_fc_xent: NULL pointer");
  const size_t bytes = (size_t)(C * B + J * C + B * J) * sizeof(float);
  if (int rc = head_smem((const void*)fc_xent_kernel, bytes)) return rc;
  fc_xent_kernel<<<(unsigned)T, kHeadThreads, bytes, (cudaStream_t)stream>>>(
      (int)B, (int)C, (int)J, 1.0f / (float)B, h4, Wfc, bfc, labels, loss, prob, dW, db, dh4);
  return launched();
}

int net_fc_xent_jvp(int64_t T, int64_t B, int64_t C, int64_t J, const float* h4, const float* h4d,
                    const float* Wfc, const float* Wd, const float* bd, const int64_t* labels,
                    const float* prob, float* dWd_acc, float* dbd_acc, float* dh4d,
                    void* stream) {
  if (T < 0 || B < 1 || C < 1 || J < 1 || T > 65535 || B * C > (1 << 24) || J > 1024)
    return fail("net_fc_xent_jvp: bad sizes");
  if (T == 0) return NET_OK;
  if (!h4 || !Wfc || !labels || !prob || !dh4d) return fail("net_fc_xent_jvp: NULL pointer");
  const size_t bytes = (size_t)(2 * C * B + 2 * J * C + 2 * B * J) * sizeof(float);
  if (int rc = head_smem((const void*)fc_xent_jvp_kernel, bytes)) return rc;
  fc_xent_jvp_kernel<<<(unsigned)T, kHeadThreads, bytes, (cudaStream_t)stream>>>(
      (int)B, (int)C, (int)J, 1.0f / (float)B, h4, h4d, Wfc, Wd, bd, labels, prob, dWd_acc,
      dbd_acc, dh4d);
  return launched();
}

int net_task_sum(int64_t T, int64_t n_leaves, const int64_t* h_offsets, const int64_t* d_offsets,
                 const float* in, float* out, void* stream) {
  if (T < 0 || n_leaves < 1 || !h_offsets || !d_offsets) return fail("net_task_sum: bad arguments");
  if (h_offsets[0] != 0) return fail("net_task_sum: offsets[0] must be 0");
  for (int64_t l = 0; l < n_leaves; ++l)
    if (h_offsets[l + 1] < h_offsets[l]) return fail("net_task_sum: offsets must be monotone");
  const int64_t n = h_offsets[n_leaves];
  if (n == 0) return NET_OK;
  if (!in || !out) return fail("net_task_sum: NULL pointer");
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  task_sum_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(T, n_leaves, d_offsets, in,
                                                                    out);
  return launched();
}

const char* net_last_error(void) { return g_err.c_str(); }
int net_abi_version(void) { return MAMLNET_ABI_VERSION; }
int64_t net_launch_count(void) { return g_launches.load(); }

}  // extern "C"
