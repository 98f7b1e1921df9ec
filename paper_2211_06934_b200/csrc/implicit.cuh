// implicit.cuh -- fused vector kernels of the implicit-gradient solvers
// (§2.2 "Implicit Gradient (IG)", P:161:
// conjugate gradient (iMAML) and Neumann series).
//
// The matrix-vector product is the caller's (a Hessian- or Jacobian-vector
// product from autograd); everything else of a CG iteration is fused into
// three passes over HBM with device-resident scalars, so the solver never
// synchronises with the host:
//   CG_INIT : r = b - Ax0 (Ax0 NULL -> r = b), p = r;  rr = r.r
//   CG_ALPHA: pAp = p.Ap;  alpha = rr / pAp
//   CG_UPD  : x += alpha p; r -= alpha Ap;  rr_new = r.r;  beta = rr_new / rr
//   CG_DIR  : p = r + beta p
// Dot products: fp64 per-thread partials, xor-shuffle, per-block partial in
// the workspace, last block sums in block order (deterministic) and updates
// the scalar state, like the optimizer reductions.
// Neumann: v -= alpha Av ; x += v  (one pass, no reduction).
#pragma once
#include <stdint.h>

#include "step_kernel.cuh"

namespace dopt {

// device scalar state of one CG solve (caller-owned double[8])
enum CgSlot { CG_RR = 0, CG_PAP = 1, CG_ALPHA = 2, CG_BETA = 3, CG_RR0 = 4, CG_ITERS = 5 };
enum CgMode { CG_INIT = 0, CG_ALPHA_MODE = 1, CG_UPD = 2, CG_DIR = 3 };

struct CgArgs {
  int64_t n;
  float* x;
  float* r;
  float* p;
  const float* Ap;
  const float* b;
  const float* Ax0;
  double* state;
  double* partials;
  unsigned int* counter;
};

template <int MODE>
__device__ __forceinline__ void cg_elem(const CgArgs& a, int64_t i, double alpha, double beta,
                                        double& acc) {
  if (MODE == CG_INIT) {
    const float r = a.Ax0 ? a.b[i] - a.Ax0[i] : a.b[i];
    a.r[i] = r;
    a.p[i] = r;
    acc += (double)r * r;
  } else if (MODE == CG_ALPHA_MODE) {
    acc += (double)a.p[i] * (double)a.Ap[i];
  } else if (MODE == CG_UPD) {
    const float al = (float)alpha;
    a.x[i] = a.x[i] + al * a.p[i];
    const float r = a.r[i] - al * a.Ap[i];
    a.r[i] = r;
    acc += (double)r * r;
  } else {
    a.p[i] = a.r[i] + (float)beta * a.p[i];
  }
}

template <int MODE>
__device__ __forceinline__ void cg_vec(const CgArgs& a, int64_t v, double alpha, double beta,
                                       double& acc) {
  float x[4], r[4], p[4], q[4];
  const float al = (float)alpha, be = (float)beta;
  if (MODE == CG_INIT) {
    load4(a.b, v, r);
    if (a.Ax0) {
      load4(a.Ax0, v, q);
#pragma unroll
      for (int e = 0; e < 4; ++e) r[e] -= q[e];
    }
    store4(a.r, v, r);
    store4(a.p, v, r);
#pragma unroll
    for (int e = 0; e < 4; ++e) acc += (double)r[e] * r[e];
  } else if (MODE == CG_ALPHA_MODE) {
    load4(a.p, v, p);
    load4(a.Ap, v, q);
#pragma unroll
    for (int e = 0; e < 4; ++e) acc += (double)p[e] * (double)q[e];
  } else if (MODE == CG_UPD) {
    load4(a.x, v, x);
    load4(a.r, v, r);
    load4(a.p, v, p);
    load4(a.Ap, v, q);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      x[e] = x[e] + al * p[e];
      r[e] = r[e] - al * q[e];
      acc += (double)r[e] * r[e];
    }
    store4(a.x, v, x);
    store4(a.r, v, r);
  } else {
    load4(a.r, v, r);
    load4(a.p, v, p);
#pragma unroll
    for (int e = 0; e < 4; ++e) p[e] = r[e] + be * p[e];
    store4(a.p, v, p);
  }
}

template <int MODE>
__global__ void __launch_bounds__(kBlock) cg_kernel(const CgArgs a) {
  pdl_wait();
  const double alpha = (MODE == CG_UPD) ? a.state[CG_ALPHA] : 0.0;
  const double beta = (MODE == CG_DIR) ? a.state[CG_BETA] : 0.0;
  double acc = 0.0;
  const int64_t nvec = a.n >> 2, nthreads = (int64_t)gridDim.x * kBlock;
  for (int64_t v = (int64_t)blockIdx.x * kBlock + threadIdx.x; v < nvec; v += nthreads)
    cg_vec<MODE>(a, v, alpha, beta, acc);
  const int64_t i = (nvec << 2) + threadIdx.x;
  if (blockIdx.x == gridDim.x - 1 && i < a.n) cg_elem<MODE>(a, i, alpha, beta, acc);
  if (MODE == CG_DIR) return;
  __shared__ double sm[1][kWarps];
  double accv[1] = {acc};
  block_sum<1>(accv, sm);
  if (threadIdx.x == 0) a.partials[blockIdx.x] = accv[0];
  if (last_block(a.counter, gridDim.x)) {
    double s[1] = {0.0};
    for (int64_t b = threadIdx.x; b < gridDim.x; b += kBlock) s[0] += __ldcg(&a.partials[b]);
    block_sum<1>(s, sm);
    if (threadIdx.x == 0) {
      double* st = a.state;
      if (MODE == CG_INIT) {
        st[CG_RR] = s[0];
        st[CG_RR0] = s[0];
        st[CG_ITERS] = 0.0;
      } else if (MODE == CG_ALPHA_MODE) {
        st[CG_PAP] = s[0];
        st[CG_ALPHA] = s[0] == 0.0 ? 0.0 : st[CG_RR] / s[0];
      } else {
        st[CG_BETA] = st[CG_RR] == 0.0 ? 0.0 : s[0] / st[CG_RR];
        st[CG_RR] = s[0];
        st[CG_ITERS] += 1.0;
      }
      *a.counter = 0u;
    }
  }
}

__global__ void __launch_bounds__(kBlock) neumann_kernel(int64_t n, float* v, const float* Av,
                                                         float* x, float alpha) {
  pdl_wait();
  const int64_t nvec = n >> 2, nthreads = (int64_t)gridDim.x * kBlock;
  for (int64_t k = (int64_t)blockIdx.x * kBlock + threadIdx.x; k < nvec; k += nthreads) {
    float vv[4], q[4], xx[4];
    load4(v, k, vv);
    load4(Av, k, q);
    load4(x, k, xx);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      vv[e] = vv[e] - alpha * q[e];
      xx[e] = xx[e] + vv[e];
    }
    store4(v, k, vv);
    store4(x, k, xx);
  }
  const int64_t i = (nvec << 2) + threadIdx.x;
  if (blockIdx.x == gridDim.x - 1 && i < n) {
    v[i] = v[i] - alpha * Av[i];
    x[i] = x[i] + v[i];
  }
}

}  // namespace dopt
