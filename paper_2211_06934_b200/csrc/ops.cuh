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
// Raw MUFU approximations (rcp.approx / rsqrt.approx, ftz on the MUFU
// operand only): branch-free, no denormal fix-up sequences. Operands below
// FLT_MIN take the zero branch of the Z6/Z7 conventions (s or d treated as
// 0); such an s is < 1e-19, 11 orders below eps, so only eps = 0 can see it.
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
constexpr float kFltMin = 1.17549435e-38f;
__device__ __forceinline__ float safe_rcp(float x) { return x >= kFltMin ? rcp_approx(x) : 0.f; }
__device__ __forceinline__ float ct_sqrt(float x) { return x >= kFltMin ? x * rsqrt_approx(x) : 0.f; }
__device__ __forceinline__ float ct_div(float a, float b) { return a * safe_rcp(b); }
__device__ __forceinline__ float rsqrt_or_zero(float x) { return x >= kFltMin ? rsqrt_approx(x) : 0.f; }
#endif

// Every op exposes apply() on compute-type scalars (so the variants below
// can feed it a transformed gradient) and set_lr() (per-leaf learning rates:
// the leaf kernel re-targets a copy of the op once per tile).

// ------------------------------------------------------------------ Adam
template <class CT_>
struct AdamFwd {
  typedef CT_ CT;
  static constexpr int NIN = 4, NOUT = 4, NH = 0;  // in: g m v params ; out: u m' v' params'
  __host__ __device__ static constexpr bool in_state(int i) { return i == 1 || i == 2; }
  __host__ __device__ static constexpr bool out_state(int i) { return i == 1 || i == 2; }
  CT b1, om1, b2, om2, ibc1, ibc2, lr, eps, eps_root;

  __device__ __forceinline__ void set_lr(CT l) { lr = l; }
  // (u, m', v') of gradient g
  __device__ __forceinline__ void apply(CT g, CT m, CT v, CT& u, CT& m1, CT& v1) const {
    m1 = b1 * m + om1 * g;
    v1 = b2 * v + om2 * (g * g);
    const CT s = ct_sqrt(v1 * ibc2 + eps_root);
    const CT d = s + eps;
    u = (-lr * (m1 * ibc1)) * safe_rcp(d);  // Z7: u = 0 when d = 0
  }
  __device__ __forceinline__ void operator()(const float (&x)[NIN], CT (&y)[NOUT], CT*,
                                             bool) const {
    apply(x[0], x[1], x[2], y[0], y[1], y[2]);
    y[3] = CT(x[3]) + y[0];
  }
};

template <class CT_>
struct AdamBwd {
  typedef CT_ CT;
  static constexpr int NIN = 6, NOUT = 3, NH = 4;  // in: g m v du dm1 dv1 ; out: dg dm dv
  __host__ __device__ static constexpr bool in_state(int i) { return i == 1 || i == 2; }
  __host__ __device__ static constexpr bool out_state(int) { return false; }
  // host-precomputed (abi.cu): A=(1-b1)/bc1, C=(1-b2)/bc2, b1ibc1=b1/bc1,
  // b2ibc2=b2/bc2, Aeps=A*eps, kM0=b1/bc1, kV0=b2/(2*bc2); set_lr derives
  // kM=kM0*lr, kV=kV0*lr, hlr=lr/2
  CT b1, om1, b2, two_om2, A, C, b1ibc1, b2ibc2, eps_root, lr, eps, Aeps, kM, kV, hlr;
  CT kM0, kV0, K1, K2, K3, K4;

  __device__ __forceinline__ void set_lr(CT l) {
    lr = l;
    kM = kM0 * l;
    kV = kV0 * l;
    hlr = CT(0.5) * l;
  }
  // dg, dm, dv of gradient g; hyper terms (lr, b1, b2, eps) into h
  __device__ __forceinline__ void apply(CT g, CT m, CT v, CT du, CT dm1, CT dv1, CT& dg, CT& dm,
                                        CT& dv, CT* h, bool want_hp) const {
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
    dg = om1 * dm1 + two_om2 * g * dv1 - (lr * T) * (Aeps + (A * Q - P * C * g) * rs);
    dm = b1 * dm1 - kM * R;                  // b1 (dm1 - du lr/(bc1 d))
    dv = b2 * dv1 + kV * U;                  // b2 (dv1 + du lr mhat/(2 s bc2 d^2))
    if (want_hp) {
      h[0] -= mhat * R;                                         // lr
      h[1] += dm1 * (m - g) - (lr * R) * (m * K1 - g * K2);     // b1
      h[2] += dv1 * (v - gg) + (hlr * U) * (v * K3 - gg * K4);  // b2
      h[3] += lr * (mhat * T);                                  // eps
    }
  }
  __device__ __forceinline__ void operator()(const float (&x)[NIN], CT (&y)[NOUT], CT* h,
                                             bool want_hp) const {
    apply(x[0], x[1], x[2], x[3], x[4], x[5], y[0], y[1], y[2], h, want_hp);
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

  __device__ __forceinline__ void set_lr(CT l) { lr = l; }
  __device__ __forceinline__ void apply(CT g, CT v, CT& u, CT& v1) const {
    v1 = alpha * v + oma * (g * g);
    const CT d = ct_sqrt(v1) + eps;
    u = (-lr * g) * safe_rcp(d);  // Z7: u = 0 when d = 0
  }
  __device__ __forceinline__ void operator()(const float (&x)[NIN], CT (&y)[NOUT], CT*,
                                             bool) const {
    apply(x[0], x[1], y[0], y[1]);
    y[2] = CT(x[2]) + y[0];
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

  __device__ __forceinline__ void set_lr(CT l) {
    lr = l;
    hlr = CT(0.5) * l;
  }
  // dg, dv; hyper terms (lr, alpha, eps)
  __device__ __forceinline__ void apply(CT g, CT v, CT du, CT dv1, CT& dg, CT& dv, CT* h,
                                        bool want_hp) const {
    const CT gg = g * g;
    const CT s2 = alpha * v + oma * gg;
    const CT rs = rsqrt_or_zero(s2);
    const CT d = s2 * rs + eps;
    const CT rd = safe_rcp(d);
    const CT R = du * rd;                   // du/d
    const CT T = R * rd;                    // du/d^2
    const CT V = dv1 + hlr * (g * T) * rs;  // dv1 + du lr g/(2 s d^2)
    dg = two_oma * g * dv1 - (lr * T) * (eps + alpha * v * rs);
    dv = alpha * V;
    if (want_hp) {
      h[0] -= g * R;
      h[1] += V * (v - gg);
      h[2] += lr * (g * T);
    }
  }
  __device__ __forceinline__ void operator()(const float (&x)[NIN], CT (&y)[NOUT], CT* h,
                                             bool want_hp) const {
    apply(x[0], x[1], x[2], x[3], y[0], y[1], h, want_hp);
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

  __device__ __forceinline__ void set_lr(CT l) { lr = l; }
  __device__ __forceinline__ void apply(CT g, CT b, CT& u, CT& b1) const {
    b1 = mu * b + g;
    u = nesterov ? -lr * (g + mu * b1) : -lr * b1;
  }
  __device__ __forceinline__ void operator()(const float (&x)[NIN], CT (&y)[NOUT], CT*,
                                             bool) const {
    apply(x[0], x[1], y[0], y[1]);
    y[2] = CT(x[2]) + y[0];
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

  __device__ __forceinline__ void set_lr(CT l) { lr = l; }
  // dg, db; hyper terms (lr, mu)
  __device__ __forceinline__ void apply(CT g, CT b, CT du, CT db1, CT& dg, CT& db, CT* h,
                                        bool want_hp) const {
    const CT b1 = mu * b + g;
    if (nesterov) {
      const CT B = db1 - lr * mu * du;
      dg = B - lr * du;
      db = mu * B;
      if (want_hp) {
        h[0] += (-du * (g + mu * b1));
        h[1] += (B * b - du * lr * b1);
      }
    } else {
      const CT B = db1 - lr * du;
      dg = B;
      db = mu * B;
      if (want_hp) {
        h[0] += (-du * b1);
        h[1] += (B * b);
      }
    }
  }
  __device__ __forceinline__ void operator()(const float (&x)[NIN], CT (&y)[NOUT], CT* h,
                                             bool want_hp) const {
    apply(x[0], x[1], x[2], x[3], y[0], y[1], h, want_hp);
  }
};

// ------------------------------------------- optimizer variants (NEXT-1)
// Weight decay, maximize and per-leaf lr (reading N1, torch.optim
// semantics): g~ = (maximize ? -g : g) + wd theta (L2), or for Adam with
// `decoupled` (AdamW) u += -lr wd theta instead. theta is the params input.
// The VJP chains the base op's VJP through g~ and adds the theta cotangent
// through the decay (`dtheta`, NOT including the identity of a fused apply)
// and the weight-decay hyper-gradient (last hyper slot).
template <class Base>
struct ExCommon {
  typedef typename Base::CT CT;
  Base base;
  CT wd;
  int decoupled, maximize;
  __device__ __forceinline__ void set_lr(CT l) { base.set_lr(l); }
  __device__ __forceinline__ CT gtilde(CT g, CT th) const {
    const CT gm = maximize ? -g : g;
    return decoupled ? gm : gm + wd * th;
  }
};

template <class CT_>
struct AdamFwdEx : ExCommon<AdamFwd<CT_>> {
  typedef CT_ CT;
  static constexpr int NIN = 4, NOUT = 4, NH = 0;  // in: g m v theta ; out: u m' v' theta'
  __host__ __device__ static constexpr bool in_state(int i) { return i == 1 || i == 2; }
  __host__ __device__ static constexpr bool out_state(int i) { return i == 1 || i == 2; }
  __device__ __forceinline__ void operator()(const float (&x)[NIN], CT (&y)[NOUT], CT*,
                                             bool) const {
    const CT th = x[3];
    this->base.apply(this->gtilde(x[0], th), x[1], x[2], y[0], y[1], y[2]);
    if (this->decoupled) y[0] -= (this->base.lr * this->wd) * th;
    y[3] = th + y[0];
  }
};

template <class CT_>
struct AdamBwdEx : ExCommon<AdamBwd<CT_>> {
  typedef CT_ CT;
  // in: g m v theta du dm1 dv1 ; out: dg dm dv dtheta ; hyper: lr b1 b2 eps wd
  static constexpr int NIN = 7, NOUT = 4, NH = 5;
  __host__ __device__ static constexpr bool in_state(int i) { return i == 1 || i == 2; }
  __host__ __device__ static constexpr bool out_state(int) { return false; }
  __device__ __forceinline__ void operator()(const float (&x)[NIN], CT (&y)[NOUT], CT* h,
                                             bool want_hp) const {
    const CT th = x[3], du = x[4];
    CT dgt;
    this->base.apply(this->gtilde(x[0], th), x[1], x[2], du, x[5], x[6], dgt, y[1], y[2], h,
                     want_hp);
    y[0] = this->maximize ? -dgt : dgt;
    const CT lr = this->base.lr;
    if (this->decoupled) {
      y[3] = -(lr * this->wd) * du;
      if (want_hp) {
        h[0] -= du * (this->wd * th);
        h[4] -= du * (lr * th);
      }
    } else {
      y[3] = this->wd * dgt;
      if (want_hp) h[4] += dgt * th;
    }
  }
};

template <class CT_>
struct RmsFwdEx : ExCommon<RmsFwd<CT_>> {
  typedef CT_ CT;
  static constexpr int NIN = 3, NOUT = 3, NH = 0;  // in: g v theta ; out: u v' theta'
  __host__ __device__ static constexpr bool in_state(int i) { return i == 1; }
  __host__ __device__ static constexpr bool out_state(int i) { return i == 1; }
  __device__ __forceinline__ void operator()(const float (&x)[NIN], CT (&y)[NOUT], CT*,
                                             bool) const {
    const CT th = x[2];
    this->base.apply(this->gtilde(x[0], th), x[1], y[0], y[1]);
    y[2] = th + y[0];
  }
};

template <class CT_>
struct RmsBwdEx : ExCommon<RmsBwd<CT_>> {
  typedef CT_ CT;
  // in: g v theta du dv1 ; out: dg dv dtheta ; hyper: lr alpha eps wd
  static constexpr int NIN = 5, NOUT = 3, NH = 4;
  __host__ __device__ static constexpr bool in_state(int i) { return i == 1; }
  __host__ __device__ static constexpr bool out_state(int) { return false; }
  __device__ __forceinline__ void operator()(const float (&x)[NIN], CT (&y)[NOUT], CT* h,
                                             bool want_hp) const {
    const CT th = x[2];
    CT dgt;
    this->base.apply(this->gtilde(x[0], th), x[1], x[3], x[4], dgt, y[1], h, want_hp);
    y[0] = this->maximize ? -dgt : dgt;
    y[2] = this->wd * dgt;
    if (want_hp) h[3] += dgt * th;
  }
};

template <class CT_>
struct SgdFwdEx : ExCommon<SgdFwd<CT_>> {
  typedef CT_ CT;
  static constexpr int NIN = 3, NOUT = 3, NH = 0;  // in: g b theta ; out: u b' theta'
  __host__ __device__ static constexpr bool in_state(int i) { return i == 1; }
  __host__ __device__ static constexpr bool out_state(int i) { return i == 1; }
  __device__ __forceinline__ void operator()(const float (&x)[NIN], CT (&y)[NOUT], CT*,
                                             bool) const {
    const CT th = x[2];
    this->base.apply(this->gtilde(x[0], th), x[1], y[0], y[1]);
    y[2] = th + y[0];
  }
};

template <class CT_>
struct SgdBwdEx : ExCommon<SgdBwd<CT_>> {
  typedef CT_ CT;
  // in: g b theta du db1 ; out: dg db dtheta ; hyper: lr mu wd
  static constexpr int NIN = 5, NOUT = 3, NH = 3;
  __host__ __device__ static constexpr bool in_state(int i) { return i == 1; }
  __host__ __device__ static constexpr bool out_state(int) { return false; }
  __device__ __forceinline__ void operator()(const float (&x)[NIN], CT (&y)[NOUT], CT* h,
                                             bool want_hp) const {
    const CT th = x[2];
    CT dgt;
    this->base.apply(this->gtilde(x[0], th), x[1], x[3], x[4], dgt, y[1], h, want_hp);
    y[0] = this->maximize ? -dgt : dgt;
    y[2] = this->wd * dgt;
    if (want_hp) h[2] += dgt * th;
  }
};

// -------------------------- fused inner-loss glue (NEXT-2, C3 sweep step)
// The synthetic inner loss L_in = 1/2 sum a (theta - phi)^2 (DESIGN.md input
// recipe, C3) folded into the unrolled Adam step so one pass does what the
// glue kernels + the plain step do in two:
//   forward  (in: a theta phi m v ; out: g m' v' theta'):
//     g = a (theta - phi) (saved for the reverse), Adam step on g, theta' = theta + u
//   reverse  (in: a g m v theta_bar dm1 dv1 phi_bar ; out: dm dv theta_bar' phi_bar'):
//     the Adam VJP with du = theta_bar (the cotangent of theta' through the
//     fused apply), then theta_bar' = theta_bar + a dg (apply identity + H^T dg,
//     H = diag a) and phi_bar' = phi_bar - a dg; dg itself is never stored.
template <class CT_>
struct AdamQuadFwd {
  typedef CT_ CT;
  static constexpr int NIN = 5, NOUT = 4, NH = 0;
  __host__ __device__ static constexpr bool in_state(int i) { return i == 3 || i == 4; }
  __host__ __device__ static constexpr bool out_state(int i) { return i == 1 || i == 2; }
  AdamFwd<CT> base;
  __device__ __forceinline__ void set_lr(CT l) { base.set_lr(l); }
  __device__ __forceinline__ void operator()(const float (&x)[NIN], CT (&y)[NOUT], CT*,
                                             bool) const {
    const CT th = x[1];
    const CT g = CT(x[0]) * (th - CT(x[2]));
    CT u;
    base.apply(g, x[3], x[4], u, y[1], y[2]);
    y[0] = g;
    y[3] = th + u;
  }
};

template <class CT_>
struct AdamQuadRev {
  typedef CT_ CT;
  static constexpr int NIN = 8, NOUT = 4, NH = 4;
  __host__ __device__ static constexpr bool in_state(int i) { return i == 2 || i == 3; }
  __host__ __device__ static constexpr bool out_state(int) { return false; }
  AdamBwd<CT> base;
  __device__ __forceinline__ void set_lr(CT l) { base.set_lr(l); }
  __device__ __forceinline__ void operator()(const float (&x)[NIN], CT (&y)[NOUT], CT* h,
                                             bool want_hp) const {
    const CT a = x[0], thb = x[4];
    CT dg;
    base.apply(x[1], x[2], x[3], thb, x[5], x[6], dg, y[0], y[1], h, want_hp);
    const CT adg = a * dg;
    y[2] = thb + adg;
    y[3] = CT(x[7]) - adg;
  }
};

// -------------------------- RMSProp centred / momentum (NEXT-1, reading N4)
// torch.optim.RMSprop semantics on g~ = (maximize ? -g : g) + wd theta:
//   v' = alpha v + (1-alpha) g~^2;  centred: a' = alpha a + (1-alpha) g~,
//   q = v' - a'^2 (else a' = a, q = v');  d = sqrt(q) + eps;  w = g~/d;
//   b' = mu b + w;  u = -lr b'.
// Reduced VJP (no cancellation between the w path and the q path), with
// B = db1 - lr du, T = B/d^2, r = sqrt(q):
//   dg~ = 2(1-alpha) g~ dv1 + (1-alpha) da1 [centred]
//         + T (eps + alpha (v - a a1) / r)          (a a1 := 0 if not centred)
//   qbar = -g~ T/(2 r),  dv = alpha (dv1 + qbar),  da = alpha (da1 - 2 a1 qbar)
//   db = mu B; hyper: lr -du b1, alpha (dv1+qbar)(v-g~^2) + A (a-g~), eps -g~ T,
//   mu B b, wd dg~ theta. sqrt(q <= 0) := 0 and its adjoint := 0.
template <class CT_>
struct RmsCmFwd {
  typedef CT_ CT;
  // in: g v a b theta ; out: u v' a' b' theta'
  static constexpr int NIN = 5, NOUT = 5, NH = 0;
  __host__ __device__ static constexpr bool in_state(int i) { return i >= 1 && i <= 3; }
  __host__ __device__ static constexpr bool out_state(int i) { return i >= 1 && i <= 3; }
  CT alpha, oma, lr, eps, mu, wd;
  int centered, maximize;

  __device__ __forceinline__ void set_lr(CT l) { lr = l; }
  __device__ __forceinline__ void operator()(const float (&x)[NIN], CT (&y)[NOUT], CT*,
                                             bool) const {
    const CT th = x[4];
    const CT gt = (maximize ? -CT(x[0]) : CT(x[0])) + wd * th;
    const CT v1 = alpha * CT(x[1]) + oma * (gt * gt);
    const CT a1 = centered ? alpha * CT(x[2]) + oma * gt : CT(x[2]);
    const CT q = centered ? v1 - a1 * a1 : v1;
    const CT d = q * rsqrt_or_zero(q) + eps;
    const CT b1 = mu * CT(x[3]) + gt * safe_rcp(d);
    y[0] = -lr * b1;
    y[1] = v1;
    y[2] = a1;
    y[3] = b1;
    y[4] = th + y[0];
  }
};

template <class CT_>
struct RmsCmBwd {
  typedef CT_ CT;
  // in: g v a b theta du dv1 da1 db1 ; out: dg dv da db dtheta
  // hyper: lr alpha eps mu wd
  static constexpr int NIN = 9, NOUT = 5, NH = 5;
  __host__ __device__ static constexpr bool in_state(int i) { return i >= 1 && i <= 3; }
  __host__ __device__ static constexpr bool out_state(int) { return false; }
  CT alpha, oma, lr, eps, mu, wd;  // every field set by abi.cu fill_rms_cm
  int centered, maximize;

  __device__ __forceinline__ void set_lr(CT l) { lr = l; }
  __device__ __forceinline__ void operator()(const float (&x)[NIN], CT (&y)[NOUT], CT* h,
                                             bool want_hp) const {
    const CT v = x[1], a = x[2], b = x[3], th = x[4], du = x[5], dv1 = x[6], da1 = x[7];
    const CT gt = (maximize ? -CT(x[0]) : CT(x[0])) + wd * th;
    const CT gg = gt * gt;
    const CT v1 = alpha * v + oma * gg;
    const CT a1 = centered ? alpha * a + oma * gt : a;
    const CT q = centered ? v1 - a1 * a1 : v1;
    const CT rs = rsqrt_or_zero(q);          // 1/r  (0 at q <= 0)
    const CT rd = safe_rcp(q * rs + eps);    // 1/d  (0 at d = 0)
    const CT B = CT(x[8]) - lr * du;         // total cotangent of b'
    const CT T = B * rd * rd;
    const CT qb = CT(-0.5) * (gt * T) * rs;  // cotangent of q
    const CT V = dv1 + qb;
    const CT A = centered ? da1 - CT(2) * a1 * qb : da1;
    const CT dgt = CT(2) * oma * gt * dv1 + (centered ? oma * da1 : CT(0)) +
                   T * (eps + alpha * (v - (centered ? a * a1 : CT(0))) * rs);
    y[0] = maximize ? -dgt : dgt;
    y[1] = alpha * V;
    y[2] = centered ? alpha * A : A;
    y[3] = mu * B;
    y[4] = wd * dgt;
    if (want_hp) {
      h[0] -= du * (mu * b + gt * rd);                          // lr
      h[1] += V * (v - gg) + (centered ? A * (a - gt) : CT(0));  // alpha
      h[2] -= gt * T;                                            // eps
      h[3] += B * b;                                             // momentum
      h[4] += dgt * th;                                          // weight decay
    }
  }
};

}  // namespace dopt
