// oracle/oracle.hpp -- scalar reference for the differentiable optimizer step.
//
// TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load, call or link
// anything under oracle/. The product path (paper_2211_06934_b200/) never
// does, and shares no code, header, table or constant with this file.
//
// What this computes (PAPER.md = P:, SPEC.md = S:, SURVEY.md §8(c) readings Z*):
//   * The paper names the accelerated, differentiable optimizers "SGD, RMSProp,
//     Adam" (§1 contribution (2)(i)) and says their forward and backward
//     are written by hand (§2.3 "CPU/GPU-accelerated optimizers"). It
//     prints no formula; the recurrences are the standard ones quoted by
//     S:188 (adam), S:196-204 (sgd), S:206 (rmsprop) -- reading Z1.
//   * The backward is the vector-Jacobian product of the step map
//         (g, state, hyper) -> (u, state')
//     written here as plain reverse-mode: one adjoint per intermediate of the
//     forward, in reverse order. No symbolic reduction is applied on purpose,
//     so that this file and the CUDA kernels are two independent derivations.
//   * 0/0 handling ("explicitly canceling some 0/0 cases"): reading Z6 --
//     if s = sqrt(.) == 0 the adjoint through the sqrt is 0; reading Z7 -- if
//     d = s + eps == 0 the update is 0 and every adjoint through 1/d is 0.
//
// Everything is templated on the scalar T so that the same text runs in
// double (the oracle), long double (x87 80-bit, for parity on inputs where
// the textbook chain rule loses digits) and std::complex<double>
// (complex-step pins of the VJP against the forward).
#pragma once
#include <cmath>
#include <complex>
#include <cstdint>

namespace oracle {

// Real part, for the branch tests at the singular points.
inline double re(double x) { return x; }
inline double re(long double x) { return (double)x; }
inline double re(const std::complex<double>& x) { return x.real(); }

// b^t by repeated multiplication: exact integer powers, S:251 (DESIGN
// DECISIONS: "bias-correction uses exact powers b1^t, b2^t").
template <class T>
T ipow(T b, int64_t t) {
  T r = T(1);
  for (int64_t i = 0; i < t; ++i) r = r * b;
  return r;
}

template <class T>
T tsqrt(const T& x) {
  using std::sqrt;
  return sqrt(x);
}

// ---------------------------------------------------------------- Adam ----
// m <- b1 m + (1-b1) g ; v <- b2 v + (1-b2) g^2 ;
//        mhat = m/(1-b1^t) ; vhat = v/(1-b2^t) ; u = -lr mhat/(sqrt(vhat)+eps)
// eps_root (reading Z4) is added under the sqrt; default 0 reproduces S:188.
// t is the 1-based step count (reading Z3; S:193 uses t=1 on the first step).
template <class T>
struct AdamHP {
  T lr, b1, b2, eps, eps_root;
};

template <class T>
struct AdamFwd {
  T u, m1, v1;
};

template <class T>
AdamFwd<T> adam_fwd(T g, T m, T v, const AdamHP<T>& h, int64_t t) {
  const T one(1);
  T m1 = h.b1 * m + (one - h.b1) * g;         // S:188 first moment
  T v1 = h.b2 * v + (one - h.b2) * g * g;     // S:188 second moment
  T bc1 = one - ipow(h.b1, t);                // S:188 bias corrections
  T bc2 = one - ipow(h.b2, t);
  T mhat = m1 / bc1;
  T vhat = v1 / bc2;
  T s = tsqrt(vhat + h.eps_root);
  T d = s + h.eps;
  T u = (re(d) == 0.0) ? T(0) : -h.lr * mhat / d;  // Z7: d == 0 -> u := 0
  return {u, m1, v1};
}

template <class T>
struct AdamVjp {
  T dg, dm, dv;              // cotangents of the inputs g, m, v
  T dlr, db1, db2, deps;     // hyper-parameter cotangents (this element's term)
};

// Reverse mode over the forward graph above. Inputs du, dm1, dv1 are the
// cotangents of the outputs u, m1, v1. ("manually writing the forward
// and backward functions"; reading Z5 for which cotangents are produced.)
template <class T>
AdamVjp<T> adam_vjp(T g, T m, T v, T du, T dm1_out, T dv1_out,
                    const AdamHP<T>& h, int64_t t) {
  const T one(1), two(2);
  // ---- forward, keeping every intermediate
  T m1 = h.b1 * m + (one - h.b1) * g;
  T v1 = h.b2 * v + (one - h.b2) * g * g;
  T p1 = ipow(h.b1, t), p2 = ipow(h.b2, t);
  T bc1 = one - p1, bc2 = one - p2;
  T mhat = m1 / bc1;
  T vhat = v1 / bc2;
  T s = tsqrt(vhat + h.eps_root);
  T d = s + h.eps;
  const bool d_zero = re(d) == 0.0;   // Z7
  const bool s_zero = re(s) == 0.0;   // Z6
  // ---- reverse: u = -lr * mhat / d
  T dlr = d_zero ? T(0) : du * (-mhat / d);
  T dmhat = d_zero ? T(0) : du * (-h.lr / d);
  T dd = d_zero ? T(0) : du * (h.lr * mhat / (d * d));
  // d = s + eps
  T deps = dd;
  T ds = dd;
  // s = sqrt(vhat + eps_root)   (Z6: adjoint through sqrt at 0 is 0)
  T dvhat = s_zero ? T(0) : ds / (two * s);
  // mhat = m1 / bc1 ; vhat = v1 / bc2
  T dm1 = dm1_out + dmhat / bc1;
  T dbc1 = -dmhat * m1 / (bc1 * bc1);
  T dv1 = dv1_out + dvhat / bc2;
  T dbc2 = -dvhat * v1 / (bc2 * bc2);
  // bc = 1 - b^t  ->  d(bc)/db = -t b^(t-1)
  T tt = T((double)t);
  T db1 = -dbc1 * tt * ipow(h.b1, t - 1);
  T db2 = -dbc2 * tt * ipow(h.b2, t - 1);
  // m1 = b1 m + (1-b1) g ; v1 = b2 v + (1-b2) g^2
  db1 = db1 + dm1 * (m - g);
  db2 = db2 + dv1 * (v - g * g);
  T dm = dm1 * h.b1;
  T dv = dv1 * h.b2;
  T dg = dm1 * (one - h.b1) + dv1 * (one - h.b2) * two * g;
  return {dg, dm, dv, dlr, db1, db2, deps};
}

// ------------------------------------------------------------- RMSProp ----
// nu <- alpha nu + (1-alpha) g^2 ; u = -lr g/(sqrt(nu)+eps)
// (eps outside the sqrt, not centred, no momentum -- reading Z1).
template <class T>
struct RmsHP {
  T lr, alpha, eps;
};

template <class T>
struct RmsFwd {
  T u, v1;
};

template <class T>
RmsFwd<T> rmsprop_fwd(T g, T v, const RmsHP<T>& h) {
  const T one(1);
  T v1 = h.alpha * v + (one - h.alpha) * g * g;
  T s = tsqrt(v1);
  T d = s + h.eps;
  T u = (re(d) == 0.0) ? T(0) : -h.lr * g / d;  // Z7
  return {u, v1};
}

template <class T>
struct RmsVjp {
  T dg, dv;
  T dlr, dalpha, deps;
};

template <class T>
RmsVjp<T> rmsprop_vjp(T g, T v, T du, T dv1_out, const RmsHP<T>& h) {
  const T one(1), two(2);
  T v1 = h.alpha * v + (one - h.alpha) * g * g;
  T s = tsqrt(v1);
  T d = s + h.eps;
  const bool d_zero = re(d) == 0.0;
  const bool s_zero = re(s) == 0.0;
  // u = -lr * g / d
  T dlr = d_zero ? T(0) : du * (-g / d);
  T dg = d_zero ? T(0) : du * (-h.lr / d);
  T dd = d_zero ? T(0) : du * (h.lr * g / (d * d));
  T deps = dd;
  T ds = dd;
  T dv1 = dv1_out + (s_zero ? T(0) : ds / (two * s));  // Z6
  // v1 = alpha v + (1-alpha) g^2
  T dalpha = dv1 * (v - g * g);
  T dv = dv1 * h.alpha;
  dg = dg + dv1 * (one - h.alpha) * two * g;
  return {dg, dv, dlr, dalpha, deps};
}

// ------------------------------------------------------- SGD-momentum ----
// momentum = 0 -> u = -lr g ; else b <- mu b + g (no dampening,
// pinned by S:203: buffers 1 then 1.9) and u = -lr b ; Nesterov (Z14):
// u = -lr (g + mu b').
template <class T>
struct SgdHP {
  T lr, mu;
  int nesterov;
};

template <class T>
struct SgdFwd {
  T u, b1;
};

template <class T>
SgdFwd<T> sgd_fwd(T g, T b, const SgdHP<T>& h) {
  T b1 = h.mu * b + g;
  T u = h.nesterov ? -h.lr * (g + h.mu * b1) : -h.lr * b1;
  return {u, b1};
}

template <class T>
struct SgdVjp {
  T dg, db;
  T dlr, dmu;
};

template <class T>
SgdVjp<T> sgd_vjp(T g, T b, T du, T db1_out, const SgdHP<T>& h) {
  T b1 = h.mu * b + g;
  T dlr, dmu, dg, db1;
  if (h.nesterov) {
    // u = -lr * (g + mu * b1)
    T w = g + h.mu * b1;
    dlr = du * (-w);
    T dw = du * (-h.lr);
    dg = dw;
    dmu = dw * b1;
    db1 = db1_out + dw * h.mu;
  } else {
    // u = -lr * b1
    dlr = du * (-b1);
    dg = T(0);
    dmu = T(0);
    db1 = db1_out + du * (-h.lr);
  }
  // b1 = mu * b + g
  dmu = dmu + db1 * b;
  T db = db1 * h.mu;
  dg = dg + db1;
  return {dg, db, dlr, dmu};
}

}  // namespace oracle

// ------------------------------------------------- magnitude twins (Z10)
// Error scale for a kernel that evaluates the REDUCED forms
// in fp32: the same expression tree with every + and - replaced by |a|+|b|
// and every product by its absolute value (denominators keep their value).
// |x - ref| <= 1e-6 + 1e-5 mag(ref) is then the fp32 tolerance: it charges a
// kernel only for the conditioning of its inputs (e.g. m' = b1 m + (1-b1) g
// can cancel, and fp32 cannot even hold b1 exactly), never for a
// cancellation the reduced form removes, so a textbook-form fp32 kernel
// still fails it (verified). This is a tolerance, not a value:
// nothing here is compared against the kernels' arithmetic.
namespace oracle {

struct AdamMag {
  double u, m1, v1, dg, dm, dv, h[4];
};

// gt is the gradient value fed to the moments (denominators keep their
// values, so s and d use it); agt is its magnitude twin: |g| for the plain
// step, |g| + wd |theta| when L2 weight decay forms gt = +-g + wd theta
// (that sum's conditioning is charged like m' = b1 m + (1-b1) g in the
// numerators and, through the Lipschitz factor below, in the denominators).
inline AdamMag adam_mag2(double gt, double agt, double m, double v, double du, double dm1,
                         double dv1, const AdamHP<double>& h, int64_t t) {
  const double b1 = h.b1, b2 = h.b2, lr = std::fabs(h.lr), eps = h.eps;
  const double bc1 = 1.0 - ipow(b1, t), bc2 = 1.0 - ipow(b2, t);
  const double A = (1 - b1) / bc1, C = (1 - b2) / bc2;
  const double P = b1 * m / bc1, Q = b2 * v / bc2 + h.eps_root;
  const double s = std::sqrt(C * gt * gt + Q), d = s + eps;
  // s is sqrt(C)-Lipschitz in gt; a cancelling gt (agt > |gt|) is known to
  // the kernel only within its rounding, so 1/d and 1/s carry the factor
  // 1 + sqrt(C) (agt - |gt|) / d (or / s); exactly 1 for the plain step.
  const double ex = std::sqrt(C) * (agt - std::fabs(gt));
  const double rd = d == 0 ? 0 : (1 + ex / d) / d, rs = s == 0 ? 0 : (1 + ex / s) / s;
  const double ag = agt, g2 = agt * agt, adu = std::fabs(du);
  const double mh = A * ag + std::fabs(P);
  AdamMag r;
  r.m1 = b1 * std::fabs(m) + (1 - b1) * ag;
  r.v1 = b2 * std::fabs(v) + (1 - b2) * g2;
  r.u = lr * mh * rd;
  r.dg = (1 - b1) * std::fabs(dm1) + 2 * (1 - b2) * ag * std::fabs(dv1) +
         adu * lr * rd * rd * (A * eps + (A * std::fabs(Q) + std::fabs(P * C) * ag) * rs);
  r.dm = b1 * (std::fabs(dm1) + adu * lr * rd / bc1);
  const double w = 0.5 * lr * mh * rd * rd * rs;
  r.dv = b2 * (std::fabs(dv1) + adu * w / bc2);
  const double tt = (double)t;
  const double p1 = ipow(b1, t), p2 = ipow(b2, t);
  const double K1 = (1 - p1 + tt * p1) / (bc1 * bc1);
  const double K2 = (1 - p1 - tt * ipow(b1, t - 1) * (1 - b1)) / (bc1 * bc1);
  const double K3 = (1 - p2 + tt * p2) / (bc2 * bc2);
  const double K4 = (1 - p2 - tt * ipow(b2, t - 1) * (1 - b2)) / (bc2 * bc2);
  r.h[0] = adu * mh * rd;
  r.h[1] = std::fabs(dm1) * (std::fabs(m) + ag) +
           adu * lr * rd * (std::fabs(m * K1) + ag * std::fabs(K2));
  r.h[2] = std::fabs(dv1) * (std::fabs(v) + g2) +
           adu * w * (std::fabs(v * K3) + g2 * std::fabs(K4));
  r.h[3] = adu * lr * mh * rd * rd;
  return r;
}

inline AdamMag adam_mag(double g, double m, double v, double du, double dm1, double dv1,
                        const AdamHP<double>& h, int64_t t) {
  return adam_mag2(g, std::fabs(g), m, v, du, dm1, dv1, h, t);
}

struct RmsMag {
  double u, v1, dg, dv, h[3];
};

inline RmsMag rmsprop_mag2(double gt, double agt, double v, double du, double dv1,
                           const RmsHP<double>& h) {
  const double a = h.alpha, lr = std::fabs(h.lr), eps = h.eps;
  const double s = std::sqrt(a * v + (1 - a) * gt * gt), d = s + eps;
  const double ex = std::sqrt(1 - a) * (agt - std::fabs(gt));  // as adam_mag2
  const double rd = d == 0 ? 0 : (1 + ex / d) / d, rs = s == 0 ? 0 : (1 + ex / s) / s;
  const double ag = agt, adu = std::fabs(du);
  RmsMag r;
  r.v1 = a * std::fabs(v) + (1 - a) * ag * ag;
  r.u = lr * ag * rd;
  r.dg = 2 * (1 - a) * ag * std::fabs(dv1) + adu * lr * rd * rd * (eps + a * std::fabs(v) * rs);
  const double w = 0.5 * lr * ag * rd * rd * rs;
  r.dv = a * (std::fabs(dv1) + adu * w);
  r.h[0] = adu * ag * rd;
  r.h[1] = (std::fabs(dv1) + adu * w) * (std::fabs(v) + ag * ag);
  r.h[2] = adu * lr * ag * rd * rd;
  return r;
}

inline RmsMag rmsprop_mag(double g, double v, double du, double dv1, const RmsHP<double>& h) {
  return rmsprop_mag2(g, std::fabs(g), v, du, dv1, h);
}

struct SgdMag {
  double u, b1, dg, db, h[2];
};

inline SgdMag sgd_mag2(double agt, double b, double du, double db1, const SgdHP<double>& h) {
  const double mu = h.mu, lr = std::fabs(h.lr);
  const double ab1 = mu * std::fabs(b) + agt;
  const double adu = std::fabs(du), adb = std::fabs(db1);
  SgdMag r;
  r.b1 = ab1;
  if (h.nesterov) {
    const double B = adb + lr * mu * adu;
    r.u = lr * (agt + mu * ab1);
    r.dg = B + lr * adu;
    r.db = mu * B;
    r.h[0] = adu * (agt + mu * ab1);
    r.h[1] = B * std::fabs(b) + adu * lr * ab1;
  } else {
    const double B = adb + lr * adu;
    r.u = lr * ab1;
    r.dg = B;
    r.db = mu * B;
    r.h[0] = adu * ab1;
    r.h[1] = B * std::fabs(b);
  }
  return r;
}

inline SgdMag sgd_mag(double g, double b, double du, double db1, const SgdHP<double>& h) {
  return sgd_mag2(std::fabs(g), b, du, db1, h);
}

}  // namespace oracle

// ------------------------------------------- optimizer variants (NEXT-1)
// weight decay, maximize and per-leaf learning rates
// (learnable per-leaf lr: meta-learned hyper-parameters, MGRL P:21/P:111).
// The paper does not define these; the semantics follow torch.optim
// (reading N1 in DESIGN.md): maximize negates g first; L2 weight decay adds
// wd*theta to the (possibly negated) gradient; AdamW ("decoupled") instead
// adds -lr*wd*theta to the update. lr is the element's leaf learning rate.
// Reverse mode is again written one adjoint per forward intermediate.
namespace oracle {

template <class T>
struct ExHP {
  T wd;
  int decoupled;  // Adam only
  int maximize;
};

template <class T>
AdamFwd<T> adam_fwd_ex(T g, T m, T v, T theta, const AdamHP<T>& h, const ExHP<T>& x, int64_t t) {
  const T one(1);
  T gm = x.maximize ? -g : g;
  T gt = x.decoupled ? gm : gm + x.wd * theta;   // gradient fed to the moments
  T m1 = h.b1 * m + (one - h.b1) * gt;
  T v1 = h.b2 * v + (one - h.b2) * gt * gt;
  T bc1 = one - ipow(h.b1, t), bc2 = one - ipow(h.b2, t);
  T mhat = m1 / bc1, vhat = v1 / bc2;
  T s = tsqrt(vhat + h.eps_root);
  T d = s + h.eps;
  T u = (re(d) == 0.0) ? T(0) : -h.lr * mhat / d;
  if (x.decoupled) u = u - h.lr * x.wd * theta;
  return {u, m1, v1};
}

template <class T>
struct AdamVjpEx {
  T dg, dm, dv, dtheta;           // dtheta: through the update only (not the apply identity)
  T dlr, db1, db2, deps, dwd;
};

template <class T>
AdamVjpEx<T> adam_vjp_ex(T g, T m, T v, T theta, T du, T dm1_out, T dv1_out,
                         const AdamHP<T>& h, const ExHP<T>& x, int64_t t) {
  const T one(1);
  T gm = x.maximize ? -g : g;
  T gt = x.decoupled ? gm : gm + x.wd * theta;
  // the plain step on gt (adjoints of every intermediate, adam_vjp above)
  AdamVjp<T> c = adam_vjp<T>(gt, m, v, du, dm1_out, dv1_out, h, t);
  AdamVjpEx<T> r;
  r.dm = c.dm;
  r.dv = c.dv;
  r.db1 = c.db1;
  r.db2 = c.db2;
  r.deps = c.deps;
  r.dlr = c.dlr;
  if (x.decoupled) {
    // u += -lr * wd * theta
    r.dlr = r.dlr + du * (-x.wd * theta);
    r.dwd = du * (-h.lr * theta);
    r.dtheta = du * (-h.lr * x.wd);
  } else {
    // gt = gm + wd * theta
    r.dwd = c.dg * theta;
    r.dtheta = c.dg * x.wd;
  }
  r.dg = x.maximize ? -c.dg : c.dg;
  return r;
}

template <class T>
RmsFwd<T> rmsprop_fwd_ex(T g, T v, T theta, const RmsHP<T>& h, const ExHP<T>& x) {
  T gm = x.maximize ? -g : g;
  return rmsprop_fwd<T>(gm + x.wd * theta, v, h);
}

template <class T>
struct RmsVjpEx {
  T dg, dv, dtheta;
  T dlr, dalpha, deps, dwd;
};

template <class T>
RmsVjpEx<T> rmsprop_vjp_ex(T g, T v, T theta, T du, T dv1_out, const RmsHP<T>& h,
                           const ExHP<T>& x) {
  T gm = x.maximize ? -g : g;
  T gt = gm + x.wd * theta;
  RmsVjp<T> c = rmsprop_vjp<T>(gt, v, du, dv1_out, h);
  RmsVjpEx<T> r{x.maximize ? -c.dg : c.dg, c.dv, c.dg * x.wd, c.dlr, c.dalpha, c.deps,
                c.dg * theta};
  return r;
}

template <class T>
SgdFwd<T> sgd_fwd_ex(T g, T b, T theta, const SgdHP<T>& h, const ExHP<T>& x) {
  T gm = x.maximize ? -g : g;
  return sgd_fwd<T>(gm + x.wd * theta, b, h);
}

template <class T>
struct SgdVjpEx {
  T dg, db, dtheta;
  T dlr, dmu, dwd;
};

template <class T>
SgdVjpEx<T> sgd_vjp_ex(T g, T b, T theta, T du, T db1_out, const SgdHP<T>& h, const ExHP<T>& x) {
  T gm = x.maximize ? -g : g;
  T gt = gm + x.wd * theta;
  SgdVjp<T> c = sgd_vjp<T>(gt, b, du, db1_out, h);
  SgdVjpEx<T> r{x.maximize ? -c.dg : c.dg, c.db, c.dg * x.wd, c.dlr, c.dmu, c.dg * theta};
  return r;
}


// Magnitude twin (Z10) of the variants: the base twins at the gradient fed
// to the moments, gt = (maximize ? -g : g) + wd theta (L2 decay; AdamW keeps
// gt = +-g), with the magnitude |g| + wd |theta| in every numerator (the
// conditioning of that sum, charged like m') and gt's value in every
// denominator; plus the weight-decay terms over |.|. kind 0 adam (hp = lr,
// b1, b2, eps, eps_root), 1 rmsprop (lr, alpha, eps), 2 sgd (lr, mu,
// nesterov); s0/s1 = the state (m, v) / v / b and its cotangents. h[] =
// (lr, b1, b2, eps, wd) / (lr, alpha, eps, wd) / (lr, mu, wd).
struct ExMag {
  double u, s0, s1, dg, ds0, ds1, dtheta, h[5];
};

inline ExMag ex_mag(int kind, double g, double s0, double s1, double theta, double du,
                    double ds0, double ds1, const double* hp, const ExHP<double>& x, int64_t t) {
  const double gm = x.maximize ? -g : g, ath = std::fabs(theta), adu = std::fabs(du);
  const double lr = std::fabs(hp[0]);
  const bool l2 = !(kind == 0 && x.decoupled);
  const double gt = l2 ? gm + x.wd * theta : gm;
  const double agt = l2 ? std::fabs(g) + x.wd * ath : std::fabs(g);
  ExMag o{};
  double dgmag = 0;
  int nb = 0;  // number of base hyper slots (the wd slot follows them)
  if (kind == 0) {
    const AdamHP<double> h{hp[0], hp[1], hp[2], hp[3], hp[4]};
    const AdamMag b = adam_mag2(gt, agt, s0, s1, du, ds0, ds1, h, t);
    o.u = b.u, o.s0 = b.m1, o.s1 = b.v1, o.dg = b.dg, o.ds0 = b.dm, o.ds1 = b.dv;
    for (int k = 0; k < 4; ++k) o.h[k] = b.h[k];
    dgmag = b.dg, nb = 4;
  } else if (kind == 1) {
    const RmsHP<double> h{hp[0], hp[1], hp[2]};
    const RmsMag b = rmsprop_mag2(gt, agt, s0, du, ds0, h);
    o.u = b.u, o.s0 = b.v1, o.dg = b.dg, o.ds0 = b.dv;
    for (int k = 0; k < 3; ++k) o.h[k] = b.h[k];
    dgmag = b.dg, nb = 3;
  } else {
    const SgdHP<double> h{hp[0], hp[1], hp[2] != 0.0 ? 1 : 0};
    const SgdMag b = sgd_mag2(agt, s0, du, ds0, h);
    o.u = b.u, o.s0 = b.b1, o.dg = b.dg, o.ds0 = b.db;
    for (int k = 0; k < 2; ++k) o.h[k] = b.h[k];
    dgmag = b.dg, nb = 2;
  }
  if (l2) {  // gt = gm + wd theta: d/dwd = dgt theta, d/dtheta = dgt wd
    o.h[nb] = dgmag * ath;
    o.dtheta = x.wd * dgmag;
  } else {   // AdamW: u += -lr wd theta
    o.u += lr * x.wd * ath;
    o.h[0] += adu * x.wd * ath;
    o.h[nb] = adu * lr * ath;
    o.dtheta = adu * lr * x.wd;
  }
  return o;
}

}  // namespace oracle

// ------------------------- RMSProp, centred and/or with momentum (NEXT-1)
// SURVEY §8(f) NEXT-1 "centered and momentum RMSProp"; torch.optim.RMSprop
// semantics (reading N4), with g~ as in the variants above:
//   v' = alpha v + (1-alpha) g~^2
//   centred:  a' = alpha a + (1-alpha) g~,  q = v' - a'^2    (else a' = a, q = v')
//   d  = sqrt(q) + eps,  w = g~ / d
//   b' = mu b + w,       u = -lr b'          (mu = 0: u = -lr g~/d, the plain step)
// Conventions: sqrt(q) := 0 for q <= 0 (and its adjoint 1/(2 sqrt q) := 0);
// w := 0 when d = 0 (Z6/Z7 extended). Reverse mode: one adjoint per forward
// intermediate, in reverse order.
namespace oracle {

template <class T>
struct RmsCmHP {
  T lr, alpha, eps, mu;
  int centered;
};

template <class T>
struct RmsCmFwd {
  T u, v1, a1, b1;
};

template <class T>
RmsCmFwd<T> rmsprop_cm_fwd(T g, T v, T a, T b, T theta, const RmsCmHP<T>& h, const ExHP<T>& x) {
  const T one(1);
  const T gm = x.maximize ? -g : g;
  const T gt = gm + x.wd * theta;
  const T v1 = h.alpha * v + (one - h.alpha) * gt * gt;
  const T a1 = h.centered ? h.alpha * a + (one - h.alpha) * gt : a;
  const T q = h.centered ? v1 - a1 * a1 : v1;
  const T r = re(q) > 0.0 ? tsqrt(q) : T(0);
  const T d = r + h.eps;
  const T w = re(d) == 0.0 ? T(0) : gt / d;
  const T b1 = h.mu * b + w;
  return {-h.lr * b1, v1, a1, b1};
}

template <class T>
struct RmsCmVjp {
  T dg, dv, da, db, dtheta;  // dtheta: through the update only
  T dlr, dalpha, deps, dmu, dwd;
};

template <class T>
RmsCmVjp<T> rmsprop_cm_vjp(T g, T v, T a, T b, T theta, T du, T dv1_out, T da1_out, T db1_out,
                           const RmsCmHP<T>& h, const ExHP<T>& x) {
  const T one(1), two(2);
  // forward intermediates
  const T gm = x.maximize ? -g : g;
  const T gt = gm + x.wd * theta;
  const T v1 = h.alpha * v + (one - h.alpha) * gt * gt;
  const T a1 = h.centered ? h.alpha * a + (one - h.alpha) * gt : a;
  const T q = h.centered ? v1 - a1 * a1 : v1;
  const bool q_pos = re(q) > 0.0;
  const T r = q_pos ? tsqrt(q) : T(0);
  const T d = r + h.eps;
  const bool d_zero = re(d) == 0.0;
  const T w = d_zero ? T(0) : gt / d;
  const T b1 = h.mu * b + w;
  RmsCmVjp<T> o;
  // u = -lr * b1
  o.dlr = du * (-b1);
  const T db1 = db1_out + du * (-h.lr);
  // b1 = mu * b + w
  o.dmu = db1 * b;
  o.db = db1 * h.mu;
  const T dw = db1;
  // w = gt / d
  T dgt = d_zero ? T(0) : dw / d;
  const T dd = d_zero ? T(0) : -dw * gt / (d * d);
  // d = r + eps
  o.deps = dd;
  const T dr = dd;
  // r = sqrt(q)
  const T dq = q_pos ? dr / (two * r) : T(0);
  // q = v1 - a1^2 (centred) or v1
  const T dv1 = dv1_out + dq;
  const T da1 = h.centered ? da1_out - two * a1 * dq : da1_out;
  // a1 = alpha a + (1 - alpha) gt (centred) or a
  o.dalpha = T(0);
  if (h.centered) {
    o.dalpha = da1 * (a - gt);
    o.da = da1 * h.alpha;
    dgt = dgt + da1 * (one - h.alpha);
  } else {
    o.da = da1;
  }
  // v1 = alpha v + (1 - alpha) gt^2
  o.dalpha = o.dalpha + dv1 * (v - gt * gt);
  o.dv = dv1 * h.alpha;
  dgt = dgt + dv1 * (one - h.alpha) * two * gt;
  // gt = (maximize ? -g : g) + wd theta
  o.dwd = dgt * theta;
  o.dtheta = dgt * x.wd;
  o.dg = x.maximize ? -dgt : dgt;
  return o;
}

// Magnitude twin (Z10) of the reduced kernel forms (ops.cuh RmsCm*):
//   dg~ = 2(1-alpha) g~ dv1 + (1-alpha) da1 + B [eps + alpha (v - a a1)/r] / d^2,
//   B = db1 - lr du, qbar = -B g~/(2 r d^2), dv = alpha (dv1 + qbar),
//   da = alpha (da1 - 2 a1 qbar). Centred q = v' - a'^2 can cancel: every
// output downstream of q is scaled by kappa = (|v'| + a'^2)_mag / q.
struct RmsCmMag {
  double u, v1, a1, b1, dg, dv, da, db, dtheta, h[5];
};

inline RmsCmMag rmsprop_cm_mag(double g, double v, double a, double b, double theta, double du,
                               double dv1, double da1, double db1, const RmsCmHP<double>& h,
                               const ExHP<double>& x) {
  const double al = h.alpha, om = 1 - al, lr = std::fabs(h.lr), eps = h.eps, mu = h.mu;
  const double gt = (x.maximize ? -g : g) + x.wd * theta;
  const double agt = std::fabs(g) + x.wd * std::fabs(theta);
  const double v1 = al * v + om * gt * gt;
  const double a1 = h.centered ? al * a + om * gt : a;
  const double q = h.centered ? v1 - a1 * a1 : v1;
  const double r = q > 0 ? std::sqrt(q) : 0.0, d = r + eps;
  // r is L-Lipschitz in gt (L = sqrt(alpha (1-alpha)) centred, sqrt(1-alpha)
  // otherwise): the conditioning of a cancelling gt, as adam_mag2
  const double ex = std::sqrt(h.centered ? al * om : om) * (agt - std::fabs(gt));
  const double rd = d == 0 ? 0 : (1 + ex / d) / d, rs = r == 0 ? 0 : (1 + ex / r) / r;
  RmsCmMag o;
  o.v1 = al * std::fabs(v) + om * agt * agt;
  o.a1 = h.centered ? al * std::fabs(a) + om * agt : std::fabs(a);
  const double qmag = h.centered ? o.v1 + o.a1 * o.a1 : o.v1;
  const double k = q > 0 ? qmag / q : 1.0;
  const double w = agt * rd;
  o.b1 = k * (mu * std::fabs(b) + w);
  o.u = lr * o.b1;
  const double B = std::fabs(db1) + lr * std::fabs(du);
  const double qb = 0.5 * B * agt * rd * rd * rs;
  o.dg = k * (2 * om * agt * std::fabs(dv1) + om * std::fabs(da1) +
              B * rd * rd * (eps + al * (std::fabs(v) + std::fabs(a) * o.a1) * rs));
  o.dv = k * al * (std::fabs(dv1) + qb);
  o.da = k * al * (std::fabs(da1) + 2 * o.a1 * qb);
  o.db = mu * B;
  o.dtheta = x.wd * o.dg;
  o.h[0] = std::fabs(du) * o.b1;
  o.h[1] = k * ((std::fabs(dv1) + qb) * (std::fabs(v) + agt * agt) +
                (h.centered ? (std::fabs(da1) + 2 * o.a1 * qb) * (std::fabs(a) + agt) : 0.0));
  o.h[2] = k * B * agt * rd * rd;
  o.h[3] = B * std::fabs(b);
  o.h[4] = o.dg * std::fabs(theta);
  return o;
}

}  // namespace oracle

// ------------------------------------------------ zero-order ES (NEXT-3)
// PAPER.md §2.2 "Zero-order Differentiation (ZD)": ES optimizes the
// Gaussian smoothing f~_sigma(theta) = E_z[f(theta + sigma z)], z ~ N(0, I_d),
// whose gradient is (1/sigma) E_z[f(theta + sigma z) z]. Monte-Carlo estimate
// over n samples (the naive form of P:204), or the antithetic form of the
// cited ES literature (reading N3):
//   naive:      g = 1/(n sigma)  sum_i f(theta + sigma z_i) z_i
//   antithetic: g = 1/(2 n sigma) sum_i [f(theta + sigma z_i) - f(theta - sigma z_i)] z_i
// The noise z_ij is a counter-based draw keyed on (seed, sample i, element j)
// so that it never has to be stored (reading N3); this file implements that
// generator itself (it shares no code with the CUDA side, which implements
// the same definition). Box-Muller pairs: elements 2k and 2k+1 share one draw
//   key  = mix(seed ^ mix(i + 0x9E3779B97F4A7C15)),  w = mix(key + k)
//   u1 = ((w >> 41) + 0.5) 2^-23,  u2 = ((w & 0x7FFFFF) + 0.5) 2^-23
//   (23-bit uniforms: k + 0.5 is then exact in fp32 as well as fp64)
//   z_2k = sqrt(-2 ln u1) cos(2 pi u2),  z_2k+1 = sqrt(-2 ln u1) sin(2 pi u2)
// with mix the SplitMix64 finaliser.
namespace oracle {

inline uint64_t es_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

inline double es_normal(uint64_t seed, int64_t i, int64_t j) {
  const uint64_t key = es_mix(seed ^ es_mix((uint64_t)i + 0x9E3779B97F4A7C15ull));
  const uint64_t w = es_mix(key + (uint64_t)(j >> 1));
  const double u1 = ((double)(w >> 41) + 0.5) * (1.0 / 8388608.0);
  const double u2 = ((double)(w & 0x7FFFFFull) + 0.5) * (1.0 / 8388608.0);
  const double r = std::sqrt(-2.0 * std::log(u1)), a = 2.0 * 3.14159265358979323846 * u2;
  return (j & 1) ? r * std::sin(a) : r * std::cos(a);
}

}  // namespace oracle
