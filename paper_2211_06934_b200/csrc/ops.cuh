// ops.cuh -- per-element forward and backward of the three optimizers.
//
// PAPER.md §2.3: the optimizer is taken "as a whole", forward and
// backward are hand-written, "symbolic reduction" is applied and some 0/0
// cases are cancelled explicitly. The formulas below are the reduced forms
// of DESIGN.md "Kernel arithmetic"; they are algebraically
// identical to the textbook VJP the oracle implements, but avoid the
// cancellations that make the textbook form lose all digits in fp32:
//   Adam, with A=(1-b1)/bc1, C=(1-b2)/bc2, P=b1 m/bc1, Q=b2 v/bc2+eps_root,
//   so mhat = A g + P and s^2 = vhat + eps_root = C g^2 + Q:
//     dg = (1-b1) dm1 + 2(1-b2) g dv1 - du lr [A eps + (A Q - P C g)/s] / d^2
//     dm = b1 (dm1 - du lr/(bc1 d)),  dv = b2 (dv1 + du lr mhat/(2 s bc2 d^2))
//     dlr = -du mhat/d, deps = du lr mhat/d^2,
//     db1 = dm1 (m-g) - du (lr/d)(m K1 - g K2),
//     db2 = dv1 (v-g^2) + du lr mhat/(2 s d^2) (v K3 - g^2 K4)
//   with K1..K4 the host-computed bias-correction derivatives (abi.cu).
//   0/0 (readings Z6/Z7): 1/s := 0 when s == 0; 1/d := 0 (u := 0) when d == 0.
// Every op reads its inputs as float (fp32 arrays and bf16 state are exact
// in float) and computes in CT (float or double, opt_compute).
#pragma once
#include <stdint.h>

namespace dopt {

// Arithmetic primitives. fp64: IEEE div/sqrt. fp32: the MUFU approximations
// (rsqrt, rcp; <= 2 ulp) unless DOPT_IEEE_F32 -- the fp32 bar is 1e-5 of the
// magnitude twin, ~40x the approximation error, and the IEEE sequences cost
// issue slots in an HBM-bound loop.
__device__ __forceinline__ double safe_rcp(double x) { return x == 0.0 ? 0.0 : 1.0 / x; }
__device__ __forceinline__ double ct_sqrt(double x) { return sqrt(x); }
__device__ __forceinline__ double ct_div(double a, double b) { return a / b; }
__device__ __forceinline__ double rsqrt_or_zero(double x) { return x > 0.0 ? 1.0 / sqrt(x) : 0.0; }
#ifdef DOPT_IEEE_F32
__device__ __forceinline__ float safe_rcp(float x) { return x == 0.f ? 0.f : 1.f / x; }
__device__ __forceinline__ float ct_sqrt(float x) { return sqrtf(x); }
__device__ __forceinline__ float ct_div(float a, float b) { return a / b; }
__device__ __forceinline__ float rsqrt_or_zero(float x) { return x > 0.f ? 1.f / sqrtf(x) : 0.f; }
#else
__device__ __forceinline__ float safe_rcp(float x) { return x == 0.f ? 0.f : __fdividef(1.f, x); }
__device__ __forceinline__ float ct_sqrt(float x) { return x > 0.f ? x * rsqrtf(x) : 0.f; }
__device__ __forceinline__ float ct_div(float a, float b) { return __fdividef(a, b); }
__device__ __forceinline__ float rsqrt_or_zero(float x) { return x > 0.f ? rsqrtf(x) : 0.f; }
#endif

// ------------------------------------------------------------------ Adam
template <class CT_>
struct AdamFwd {
  typedef CT_ CT;
  static constexpr int NIN = 4, NOUT = 4, NH = 0;  // in: g m v params ; out: u m' v' params'
  __host__ __device__ static constexpr bool in_state(int i) { return i == 1 || i == 2; }
  __host__ __device__ static constexpr bool out_state(int i) { return i == 1 || i == 2; }
  CT b1, om1, b2, om2, ibc1, ibc2, lr, eps, eps_root;

  __device__ __forceinline__ void operator()(const float (&x)[NIN], CT (&y)[NOUT], CT*,
                                             bool) const {
    const CT g = x[0], m = x[1], v = x[2];
    const CT m1 = b1 * m + om1 * g;
    const CT v1 = b2 * v + om2 * (g * g);
    const CT s = ct_sqrt(v1 * ibc2 + eps_root);
    const CT d = s + eps;
    const CT u = d == CT(0) ? CT(0) : ct_div(-lr * (m1 * ibc1), d);
    y[0] = u;
    y[1] = m1;
    y[2] = v1;
    y[3] = CT(x[3]) + u;
  }
};

template <class CT_>
struct AdamBwd {
  typedef CT_ CT;
  static constexpr int NIN = 6, NOUT = 3, NH = 4;  // in: g m v du dm1 dv1 ; out: dg dm dv
  __host__ __device__ static constexpr bool in_state(int i) { return i == 1 || i == 2; }
  __host__ __device__ static constexpr bool out_state(int) { return false; }
  // host-precomputed (abi.cu): A=(1-b1)/bc1, C=(1-b2)/bc2, b1ibc1=b1/bc1,
  // b2ibc2=b2/bc2, Aeps=A*eps, kM=b1*lr/bc1, kV=b2*lr/(2*bc2), hlr=lr/2
  CT b1, om1, b2, two_om2, A, C, b1ibc1, b2ibc2, eps_root, lr, eps, Aeps, kM, kV, hlr;
  CT K1, K2, K3, K4;

  __device__ __forceinline__ void operator()(const float (&x)[NIN], CT (&y)[NOUT], CT* h,
                                             bool want_hp) const {
    const CT g = x[0], m = x[1], v = x[2], du = x[3], dm1 = x[4], dv1 = x[5];
    const CT P = b1ibc1 * m;                 // mhat = A g + P
    const CT Q = b2ibc2 * v + eps_root;      // s^2  = C g^2 + Q
    const CT gg = g * g;
    const CT mhat = A * g + P;
    const CT s2 = C * gg + Q;
    const CT rs = rsqrt_or_zero(s2);         // 1/s  (Z6: 0 at s = 0)
    const CT d = s2 * rs + eps;              // d = s + eps
    const CT rd = safe_rcp(d);               // 1/d  (Z7: 0 at d = 0)
    const CT R = du * rd;                    // du/d
    const CT T = R * rd;                     // du/d^2
    const CT U = mhat * T * rs;              // du mhat/(s d^2)
    // dg = (1-b1) dm1 + 2(1-b2) g dv1 - lr du [A eps + (A Q - P C g)/s]/d^2
    y[0] = om1 * dm1 + two_om2 * g * dv1 - (lr * T) * (Aeps + (A * Q - P * C * g) * rs);
    y[1] = b1 * dm1 - kM * R;                // b1 (dm1 - du lr/(bc1 d))
    y[2] = b2 * dv1 + kV * U;                // b2 (dv1 + du lr mhat/(2 s bc2 d^2))
    if (want_hp) {
      h[0] -= mhat * R;                                       // lr
      h[1] += dm1 * (m - g) - (lr * R) * (m * K1 - g * K2);   // b1
      h[2] += dv1 * (v - gg) + (hlr * U) * (v * K3 - gg * K4);  // b2
      h[3] += lr * (mhat * T);                                // eps
    }
  }
};

// --------------------------------------------------------------- RMSProp
template <class CT_>
struct RmsFwd {
  typedef CT_ CT;
  static constexpr int NIN = 3, NOUT = 3, NH = 0;  // in: g v params ; out: u v' params'
  __host__ __device__ static constexpr bool in_state(int i) { return i == 1; }
  __host__ __device__ static constexpr bool out_state(int i) { return i == 1; }
  CT alpha, oma, lr, eps;

  __device__ __forceinline__ void operator()(const float (&x)[NIN], CT (&y)[NOUT], CT*,
                                             bool) const {
    const CT g = x[0], v = x[1];
    const CT v1 = alpha * v + oma * (g * g);
    const CT d = ct_sqrt(v1) + eps;
    const CT u = d == CT(0) ? CT(0) : ct_div(-lr * g, d);
    y[0] = u;
    y[1] = v1;
    y[2] = CT(x[2]) + u;
  }
};

// Reduced: dg = 2(1-a) g dv1 - du lr [eps + a v / s] / d^2
template <class CT_>
struct RmsBwd {
  typedef CT_ CT;
  static constexpr int NIN = 4, NOUT = 2, NH = 3;  // in: g v du dv1 ; out: dg dv
  __host__ __device__ static constexpr bool in_state(int i) { return i == 1; }
  __host__ __device__ static constexpr bool out_state(int) { return false; }
  CT alpha, oma, two_oma, lr, eps, hlr;  // hlr = lr/2

  __device__ __forceinline__ void operator()(const float (&x)[NIN], CT (&y)[NOUT], CT* h,
                                             bool want_hp) const {
    const CT g = x[0], v = x[1], du = x[2], dv1 = x[3];
    const CT gg = g * g;
    const CT s2 = alpha * v + oma * gg;
    const CT rs = rsqrt_or_zero(s2);
    const CT d = s2 * rs + eps;
    const CT rd = safe_rcp(d);
    const CT R = du * rd;                   // du/d
    const CT T = R * rd;                    // du/d^2
    const CT V = dv1 + hlr * (g * T) * rs;  // dv1 + du lr g/(2 s d^2)
    y[0] = two_oma * g * dv1 - (lr * T) * (eps + alpha * v * rs);
    y[1] = alpha * V;
    if (want_hp) {
      h[0] -= g * R;
      h[1] += V * (v - gg);
      h[2] += lr * (g * T);
    }
  }
};

// ------------------------------------------------------------------- SGD
template <class CT_>
struct SgdFwd {
  typedef CT_ CT;
  static constexpr int NIN = 3, NOUT = 3, NH = 0;  // in: g b params ; out: u b' params'
  __host__ __device__ static constexpr bool in_state(int i) { return i == 1; }
  __host__ __device__ static constexpr bool out_state(int i) { return i == 1; }
  CT lr, mu;
  int nesterov;

  __device__ __forceinline__ void operator()(const float (&x)[NIN], CT (&y)[NOUT], CT*,
                                             bool) const {
    const CT g = x[0], b = x[1];
    const CT b1 = mu * b + g;
    const CT u = nesterov ? -lr * (g + mu * b1) : -lr * b1;
    y[0] = u;
    y[1] = b1;
    y[2] = CT(x[2]) + u;
  }
};

template <class CT_>
struct SgdBwd {
  typedef CT_ CT;
  static constexpr int NIN = 4, NOUT = 2, NH = 2;  // in: g b du db1 ; out: dg db
  __host__ __device__ static constexpr bool in_state(int i) { return i == 1; }
  __host__ __device__ static constexpr bool out_state(int) { return false; }
  CT lr, mu;
  int nesterov;

  __device__ __forceinline__ void operator()(const float (&x)[NIN], CT (&y)[NOUT], CT* h,
                                             bool want_hp) const {
    const CT g = x[0], b = x[1], du = x[2], db1 = x[3];
    const CT b1 = mu * b + g;
    if (nesterov) {
      const CT B = db1 - lr * mu * du;
      y[0] = B - lr * du;
      y[1] = mu * B;
      if (want_hp) {
        h[0] += (-du * (g + mu * b1));
        h[1] += (B * b - du * lr * b1);
      }
    } else {
      const CT B = db1 - lr * du;
      y[0] = B;
      y[1] = mu * B;
      if (want_hp) {
        h[0] += (-du * b1);
        h[1] += (B * b);
      }
    }
  }
};

}  // namespace dopt
