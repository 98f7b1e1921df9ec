// oracle/oracle.cpp -- array entry points of the scalar oracle (C ABI, ctypes).
//
// TEST INFRASTRUCTURE ONLY (see oracle.hpp): callable from tests/,
// __graft_entry__.smoke() and bench.py's CPU-baseline legs, never from the
// product package. Shares no code with paper_2211_06934_b200/.
//
// Conventions of this file (not of the product ABI):
//   * inputs are the exact fp32 values the GPU sees (or bf16 bit patterns for
//     state when state_bf16 = 1, promoted exactly: bits << 16);
//   * a NULL state input means the zero state (opt.init); a NULL
//     cotangent means a zero cotangent; a NULL output is skipped;
//   * outputs are double; prec = 0 evaluates in double, prec = 1 in long
//     double (x87 80-bit) -- SURVEY Z11: the textbook chain rule has relative
//     error ~1e-16 |g|/eps in dg, long double removes that from parity checks;
//   * hyper-gradient sums ("Sigma-reduced", north star) are summed per fixed
//     4096-element chunk (S:250 chunking), then over chunks in index order, in
//     long double; the result does not depend on the thread count;
//   * dhp_abs (optional) receives Sigma |term| per hyper-gradient, the scale
//     a tolerance on a sum of signed terms must use (reading Z10).
#include "oracle.hpp"

#include <cstdint>
#include <cstring>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

using oracle::AdamHP;
using oracle::RmsHP;
using oracle::SgdHP;
typedef std::complex<double> cd;

namespace {

int g_threads = 1;
const int64_t kChunk = 4096;

inline float bf16_to_f32(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

// Input element i of a state array (NULL -> 0).
inline double state_in(const void* p, int bf16, int64_t i) {
  if (!p) return 0.0;
  if (bf16) return (double)bf16_to_f32(((const uint16_t*)p)[i]);
  return (double)((const float*)p)[i];
}
inline double f32_in(const float* p, int64_t i) { return p ? (double)p[i] : 0.0; }
inline void put(double* p, int64_t i, double x) {
  if (p) p[i] = x;
}

// Run body(i, acc[]) for every element; acc has `nh` hyper-gradient slots.
// Per-chunk partials, then an index-ordered sum over chunks.
template <class Body>
void for_chunks(int64_t n, int nh, double* sums, double* abs_sums, Body body) {
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  std::vector<long double> part((size_t)nchunks * nh * 2, 0.0L);
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(g_threads)
#endif
  for (int64_t c = 0; c < nchunks; ++c) {
    long double* acc = &part[(size_t)c * nh * 2];
    const int64_t lo = c * kChunk, hi = (lo + kChunk < n) ? lo + kChunk : n;
    for (int64_t i = lo; i < hi; ++i) body(i, acc);
  }
  for (int k = 0; k < nh; ++k) {
    long double s = 0.0L, a = 0.0L;
    for (int64_t c = 0; c < nchunks; ++c) {
      s += part[(size_t)c * nh * 2 + k];
      a += part[(size_t)c * nh * 2 + nh + k];
    }
    if (sums) sums[k] = (double)s;
    if (abs_sums) abs_sums[k] = (double)a;
  }
}

inline void acc_term(long double* acc, int nh, int k, long double x) {
  acc[k] += x;
  acc[nh + k] += (x < 0 ? -x : x);
}

// Per-leaf sums: plain loop over leaves (P:87/S:120 flatten -> offsets).
template <class Term>
void leaf_sums(int64_t n_leaves, const int64_t* off, int nh, double* out, Term term) {
  for (int64_t l = 0; l < n_leaves; ++l) {
    std::vector<long double> s(nh, 0.0L);
    for (int64_t i = off[l]; i < off[l + 1]; ++i) term(i, s.data());
    for (int k = 0; k < nh; ++k) out[l * nh + k] = (double)s[k];
  }
}

template <class T>
AdamHP<T> adam_hp(const double* hp) {
  return {T(hp[0]), T(hp[1]), T(hp[2]), T(hp[3]), T(hp[4])};
}
template <class T>
RmsHP<T> rms_hp(const double* hp) {
  return {T(hp[0]), T(hp[1]), T(hp[2])};
}
template <class T>
SgdHP<T> sgd_hp(const double* hp) {
  return {T(hp[0]), T(hp[1]), hp[2] != 0.0 ? 1 : 0};
}

// ---------------------------------------------------------------- adam
template <class T>
void adam_fwd_arr(int64_t n, int64_t t, const double* hp, int bf, const float* g,
                  const void* m, const void* v, double* u, double* m1, double* v1) {
  const AdamHP<T> h = adam_hp<T>(hp);
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(g_threads)
#endif
  for (int64_t i = 0; i < n; ++i) {
    auto r = oracle::adam_fwd<T>(T(f32_in(g, i)), T(state_in(m, bf, i)),
                                 T(state_in(v, bf, i)), h, t);
    put(u, i, (double)r.u);
    put(m1, i, (double)r.m1);
    put(v1, i, (double)r.v1);
  }
}

template <class T>
void adam_vjp_arr(int64_t n, int64_t t, const double* hp, int bf, const float* g,
                  const void* m, const void* v, const float* du, const float* dm1,
                  const float* dv1, double* dg, double* dm, double* dv, double* dhp,
                  double* dhp_abs, int64_t n_leaves, const int64_t* off,
                  double* dhp_leaf) {
  const AdamHP<T> h = adam_hp<T>(hp);
  auto elem = [&](int64_t i) {
    return oracle::adam_vjp<T>(T(f32_in(g, i)), T(state_in(m, bf, i)),
                               T(state_in(v, bf, i)), T(f32_in(du, i)),
                               T(f32_in(dm1, i)), T(f32_in(dv1, i)), h, t);
  };
  for_chunks(n, 4, dhp, dhp_abs, [&](int64_t i, long double* acc) {
    auto r = elem(i);
    put(dg, i, (double)r.dg);
    put(dm, i, (double)r.dm);
    put(dv, i, (double)r.dv);
    acc_term(acc, 4, 0, (long double)r.dlr);
    acc_term(acc, 4, 1, (long double)r.db1);
    acc_term(acc, 4, 2, (long double)r.db2);
    acc_term(acc, 4, 3, (long double)r.deps);
  });
  if (dhp_leaf && off)
    leaf_sums(n_leaves, off, 4, dhp_leaf, [&](int64_t i, long double* s) {
      auto r = elem(i);
      s[0] += (long double)r.dlr;
      s[1] += (long double)r.db1;
      s[2] += (long double)r.db2;
      s[3] += (long double)r.deps;
    });
}

// ------------------------------------------------------------- rmsprop
template <class T>
void rms_fwd_arr(int64_t n, const double* hp, int bf, const float* g, const void* v,
                 double* u, double* v1) {
  const RmsHP<T> h = rms_hp<T>(hp);
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(g_threads)
#endif
  for (int64_t i = 0; i < n; ++i) {
    auto r = oracle::rmsprop_fwd<T>(T(f32_in(g, i)), T(state_in(v, bf, i)), h);
    put(u, i, (double)r.u);
    put(v1, i, (double)r.v1);
  }
}

template <class T>
void rms_vjp_arr(int64_t n, const double* hp, int bf, const float* g, const void* v,
                 const float* du, const float* dv1, double* dg, double* dv,
                 double* dhp, double* dhp_abs, int64_t n_leaves, const int64_t* off,
                 double* dhp_leaf) {
  const RmsHP<T> h = rms_hp<T>(hp);
  auto elem = [&](int64_t i) {
    return oracle::rmsprop_vjp<T>(T(f32_in(g, i)), T(state_in(v, bf, i)),
                                  T(f32_in(du, i)), T(f32_in(dv1, i)), h);
  };
  for_chunks(n, 3, dhp, dhp_abs, [&](int64_t i, long double* acc) {
    auto r = elem(i);
    put(dg, i, (double)r.dg);
    put(dv, i, (double)r.dv);
    acc_term(acc, 3, 0, (long double)r.dlr);
    acc_term(acc, 3, 1, (long double)r.dalpha);
    acc_term(acc, 3, 2, (long double)r.deps);
  });
  if (dhp_leaf && off)
    leaf_sums(n_leaves, off, 3, dhp_leaf, [&](int64_t i, long double* s) {
      auto r = elem(i);
      s[0] += (long double)r.dlr;
      s[1] += (long double)r.dalpha;
      s[2] += (long double)r.deps;
    });
}

// ----------------------------------------------------------------- sgd
template <class T>
void sgd_fwd_arr(int64_t n, const double* hp, int bf, const float* g, const void* b,
                 double* u, double* b1) {
  const SgdHP<T> h = sgd_hp<T>(hp);
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(g_threads)
#endif
  for (int64_t i = 0; i < n; ++i) {
    auto r = oracle::sgd_fwd<T>(T(f32_in(g, i)), T(state_in(b, bf, i)), h);
    put(u, i, (double)r.u);
    put(b1, i, (double)r.b1);
  }
}

template <class T>
void sgd_vjp_arr(int64_t n, const double* hp, int bf, const float* g, const void* b,
                 const float* du, const float* db1, double* dg, double* db,
                 double* dhp, double* dhp_abs, int64_t n_leaves, const int64_t* off,
                 double* dhp_leaf) {
  const SgdHP<T> h = sgd_hp<T>(hp);
  auto elem = [&](int64_t i) {
    return oracle::sgd_vjp<T>(T(f32_in(g, i)), T(state_in(b, bf, i)), T(f32_in(du, i)),
                              T(f32_in(db1, i)), h);
  };
  for_chunks(n, 2, dhp, dhp_abs, [&](int64_t i, long double* acc) {
    auto r = elem(i);
    put(dg, i, (double)r.dg);
    put(db, i, (double)r.db);
    acc_term(acc, 2, 0, (long double)r.dlr);
    acc_term(acc, 2, 1, (long double)r.dmu);
  });
  if (dhp_leaf && off)
    leaf_sums(n_leaves, off, 2, dhp_leaf, [&](int64_t i, long double* s) {
      auto r = elem(i);
      s[0] += (long double)r.dlr;
      s[1] += (long double)r.dmu;
    });
}

// ----------------------------------------------- K-step unrolled sweep
// SURVEY §8(a) row a9 (EG over unrolled optimisation, Listing 1
// P:124-132): synthetic inner loss L_in = 1/2 sum a_i (theta_i - phi_i)^2, so
// g = a (theta - phi), H = diag(a), dg/dphi = -diag(a); outer loss
// L_out = 1/2 ||theta_K - y||^2 (reading Z17). Forward k = 0..K-1 with step
// count t = k+1, theta_{k+1} = theta_k + u_k (apply_updates). Reverse:
// the VJP of each step in reverse order, theta_bar_k = theta_bar_{k+1} + H g_bar_k,
// phi_bar -= a g_bar_k, hyper_bar += this step's hyper cotangents.
// Every element is independent except for the shared hyper-parameters.
// kind: 0 adam (hp[5]), 1 rmsprop (hp[3]), 2 sgd (hp[3]: lr, mu, nesterov).
template <class T>
struct StepRes {
  T u, s1, s2;  // update and the new state(s)
};

template <class T>
StepRes<T> step_fwd(int kind, T g, T s1, T s2, const double* hp, int64_t t) {
  if (kind == 0) {
    auto r = oracle::adam_fwd<T>(g, s1, s2, adam_hp<T>(hp), t);
    return {r.u, r.m1, r.v1};
  } else if (kind == 1) {
    auto r = oracle::rmsprop_fwd<T>(g, s1, rms_hp<T>(hp));
    return {r.u, r.v1, T(0)};
  }
  auto r = oracle::sgd_fwd<T>(g, s1, sgd_hp<T>(hp));
  return {r.u, r.b1, T(0)};
}

template <class T>
void sweep_elem(int kind, int64_t K, const double* hp, T a, T th0, T phi, T y,
                T* phi_bar, T* th0_bar, T* hyper, T* loss, T* thK, double* bar_abs,
                double* hyper_abs) {
  std::vector<T> gk(K), s1k(K + 1), s2k(K + 1);
  T th = th0;
  s1k[0] = T(0);
  s2k[0] = T(0);
  for (int64_t k = 0; k < K; ++k) {
    gk[k] = a * (th - phi);
    auto r = step_fwd<T>(kind, gk[k], s1k[k], s2k[k], hp, k + 1);
    s1k[k + 1] = r.s1;
    s2k[k + 1] = r.s2;
    th = th + r.u;
  }
  *thK = th;
  *loss = T(0.5) * (th - y) * (th - y);
  T thb = th - y, s1b = T(0), s2b = T(0), phib = T(0);
  double babs = std::fabs((double)thb);  // Sigma |terms| of theta_bar / phi_bar
  for (int k = 0; k < 4; ++k) {
    hyper[k] = T(0);
    hyper_abs[k] = 0.0;
  }
  for (int64_t k = K - 1; k >= 0; --k) {
    T gb;
    if (kind == 0) {
      auto r = oracle::adam_vjp<T>(gk[k], s1k[k], s2k[k], thb, s1b, s2b, adam_hp<T>(hp), k + 1);
      gb = r.dg; s1b = r.dm; s2b = r.dv;
      hyper[0] = hyper[0] + r.dlr; hyper[1] = hyper[1] + r.db1;
      hyper[2] = hyper[2] + r.db2; hyper[3] = hyper[3] + r.deps;
      hyper_abs[0] += std::fabs((double)r.dlr); hyper_abs[1] += std::fabs((double)r.db1);
      hyper_abs[2] += std::fabs((double)r.db2); hyper_abs[3] += std::fabs((double)r.deps);
    } else if (kind == 1) {
      auto r = oracle::rmsprop_vjp<T>(gk[k], s1k[k], thb, s1b, rms_hp<T>(hp));
      gb = r.dg; s1b = r.dv;
      hyper[0] = hyper[0] + r.dlr; hyper[1] = hyper[1] + r.dalpha;
      hyper[2] = hyper[2] + r.deps;
      hyper_abs[0] += std::fabs((double)r.dlr); hyper_abs[1] += std::fabs((double)r.dalpha);
      hyper_abs[2] += std::fabs((double)r.deps);
    } else {
      auto r = oracle::sgd_vjp<T>(gk[k], s1k[k], thb, s1b, sgd_hp<T>(hp));
      gb = r.dg; s1b = r.db;
      hyper[0] = hyper[0] + r.dlr; hyper[1] = hyper[1] + r.dmu;
      hyper_abs[0] += std::fabs((double)r.dlr); hyper_abs[1] += std::fabs((double)r.dmu);
    }
    // theta_{k+1} = theta_k + u_k  -> identity on theta_bar, plus g_k = a (theta_k - phi)
    thb = thb + a * gb;
    phib = phib - a * gb;
    babs += std::fabs((double)(a * gb));
  }
  *bar_abs = babs;
  *phi_bar = phib;
  *th0_bar = thb;
}

}  // namespace

extern "C" {

int oracle_set_num_threads(int n) {
#ifdef _OPENMP
  g_threads = n > 0 ? n : omp_get_max_threads();
#else
  g_threads = 1;
  (void)n;
#endif
  return g_threads;
}

int oracle_has_openmp(void) {
#ifdef _OPENMP
  return 1;
#else
  return 0;
#endif
}

void oracle_adam_fwd(int64_t n, int64_t t, const double* hp, int state_bf16, int prec,
                     const float* g, const void* m, const void* v, double* u,
                     double* m1, double* v1) {
  if (prec)
    adam_fwd_arr<long double>(n, t, hp, state_bf16, g, m, v, u, m1, v1);
  else
    adam_fwd_arr<double>(n, t, hp, state_bf16, g, m, v, u, m1, v1);
}

void oracle_adam_vjp(int64_t n, int64_t t, const double* hp, int state_bf16, int prec,
                     const float* g, const void* m, const void* v, const float* du,
                     const float* dm1, const float* dv1, double* dg, double* dm,
                     double* dv, double* dhp, double* dhp_abs, int64_t n_leaves,
                     const int64_t* offsets, double* dhp_leaf) {
  if (prec)
    adam_vjp_arr<long double>(n, t, hp, state_bf16, g, m, v, du, dm1, dv1, dg, dm, dv,
                              dhp, dhp_abs, n_leaves, offsets, dhp_leaf);
  else
    adam_vjp_arr<double>(n, t, hp, state_bf16, g, m, v, du, dm1, dv1, dg, dm, dv, dhp,
                         dhp_abs, n_leaves, offsets, dhp_leaf);
}

void oracle_rmsprop_fwd(int64_t n, const double* hp, int state_bf16, int prec,
                        const float* g, const void* v, double* u, double* v1) {
  if (prec)
    rms_fwd_arr<long double>(n, hp, state_bf16, g, v, u, v1);
  else
    rms_fwd_arr<double>(n, hp, state_bf16, g, v, u, v1);
}

void oracle_rmsprop_vjp(int64_t n, const double* hp, int state_bf16, int prec,
                        const float* g, const void* v, const float* du, const float* dv1,
                        double* dg, double* dv, double* dhp, double* dhp_abs,
                        int64_t n_leaves, const int64_t* offsets, double* dhp_leaf) {
  if (prec)
    rms_vjp_arr<long double>(n, hp, state_bf16, g, v, du, dv1, dg, dv, dhp, dhp_abs,
                             n_leaves, offsets, dhp_leaf);
  else
    rms_vjp_arr<double>(n, hp, state_bf16, g, v, du, dv1, dg, dv, dhp, dhp_abs, n_leaves,
                        offsets, dhp_leaf);
}

void oracle_sgd_fwd(int64_t n, const double* hp, int state_bf16, int prec, const float* g,
                    const void* b, double* u, double* b1) {
  if (prec)
    sgd_fwd_arr<long double>(n, hp, state_bf16, g, b, u, b1);
  else
    sgd_fwd_arr<double>(n, hp, state_bf16, g, b, u, b1);
}

void oracle_sgd_vjp(int64_t n, const double* hp, int state_bf16, int prec, const float* g,
                    const void* b, const float* du, const float* db1, double* dg,
                    double* db, double* dhp, double* dhp_abs, int64_t n_leaves,
                    const int64_t* offsets, double* dhp_leaf) {
  if (prec)
    sgd_vjp_arr<long double>(n, hp, state_bf16, g, b, du, db1, dg, db, dhp, dhp_abs,
                             n_leaves, offsets, dhp_leaf);
  else
    sgd_vjp_arr<double>(n, hp, state_bf16, g, b, du, db1, dg, db, dhp, dhp_abs, n_leaves,
                        offsets, dhp_leaf);
}

// Round-to-nearest-even of a double to bf16 (reading Z9: stored bf16 state
// is RNE of the exact value). Independent bit-level implementation on the
// IEEE double: keep sign, exponent and the top 7 mantissa bits.
void oracle_bf16_rne(int64_t n, const double* x, uint16_t* out) {
  for (int64_t i = 0; i < n; ++i) {
    // exact double -> the nearest bf16 via the float grid: bf16 values are
    // floats whose low 16 bits are zero; find neighbours on that grid.
    double d = x[i];
    if (d != d) {  // NaN
      out[i] = 0x7FC0;
      continue;
    }
    float f = (float)d;  // nearest float (RNE); refine against d below
    uint32_t u;
    std::memcpy(&u, &f, 4);
    uint32_t lo = u & 0xFFFF0000u;          // truncation toward zero on the bf16 grid
    uint32_t hi = lo + 0x00010000u;         // next bf16 away from zero
    float flo, fhi;
    std::memcpy(&flo, &lo, 4);
    std::memcpy(&fhi, &hi, 4);
    double elo = d - (double)flo, ehi = (double)fhi - d;
    if (elo < 0) elo = -elo;
    if (ehi < 0) ehi = -ehi;
    uint32_t pick;
    if (elo < ehi) pick = lo;
    else if (ehi < elo) pick = hi;
    else pick = ((lo >> 16) & 1u) ? hi : lo;  // tie -> even
    out[i] = (uint16_t)(pick >> 16);
  }
}

// K-step sweep in double / long double. prec as above.
void oracle_sweep_quadratic(int kind, int64_t n, int64_t K, const double* hp, int prec,
                            const float* a, const float* theta0, const float* phi,
                            const float* y, double* phi_bar, double* theta0_bar,
                            double* hyper_bar, double* loss, double* thetaK, double* bar_abs,
                            double* hyper_abs) {
  std::vector<long double> hyp_part((size_t)((n + kChunk - 1) / kChunk + 1) * 9, 0.0L);
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(g_threads)
#endif
  for (int64_t c = 0; c < nchunks; ++c) {
    long double* acc = &hyp_part[(size_t)c * 9];
    const int64_t lo = c * kChunk, hi = (lo + kChunk < n) ? lo + kChunk : n;
    for (int64_t i = lo; i < hi; ++i) {
      if (prec) {
        long double pb, tb, h[4], l, tk;
        double ba, habs[4];
        sweep_elem<long double>(kind, K, hp, a[i], theta0[i], phi[i], y[i], &pb, &tb, h, &l, &tk, &ba,
                                habs);
        put(bar_abs, i, ba);
        for (int k = 0; k < 4; ++k) acc[5 + k] += habs[k];
        put(phi_bar, i, (double)pb);
        put(theta0_bar, i, (double)tb);
        put(thetaK, i, (double)tk);
        for (int k = 0; k < 4; ++k) acc[k] += h[k];
        acc[4] += l;
      } else {
        double pb, tb, h[4], l, tk;
        double ba, habs[4];
        sweep_elem<double>(kind, K, hp, a[i], theta0[i], phi[i], y[i], &pb, &tb, h, &l, &tk, &ba,
                           habs);
        put(bar_abs, i, ba);
        for (int k = 0; k < 4; ++k) acc[5 + k] += habs[k];
        put(phi_bar, i, pb);
        put(theta0_bar, i, tb);
        put(thetaK, i, tk);
        for (int k = 0; k < 4; ++k) acc[k] += h[k];
        acc[4] += l;
      }
    }
  }
  long double s[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t c = 0; c < nchunks; ++c)
    for (int k = 0; k < 9; ++k) s[k] += hyp_part[(size_t)c * 9 + k];
  for (int k = 0; k < 4; ++k) {
    if (hyper_bar) hyper_bar[k] = (double)s[k];
    if (hyper_abs) hyper_abs[k] = (double)s[5 + k];
  }
  if (loss) *loss = (double)s[4];
}

// ------------------------------------------------ complex-step entry points
// Forward maps in std::complex<double>. Each array is given as
// separate real and imaginary parts; a NULL imaginary part means 0.
static inline cd cin(const double* re_, const double* im_, int64_t i) {
  return cd(re_ ? re_[i] : 0.0, im_ ? im_[i] : 0.0);
}
static inline void cout_(double* re_, double* im_, int64_t i, cd x) {
  if (re_) re_[i] = x.real();
  if (im_) im_[i] = x.imag();
}

void oracle_adam_fwd_cplx(int64_t n, int64_t t, const double* hp_re, const double* hp_im,
                          const double* g_re, const double* g_im, const double* m_re,
                          const double* m_im, const double* v_re, const double* v_im,
                          double* u_re, double* u_im, double* m1_re, double* m1_im,
                          double* v1_re, double* v1_im) {
  AdamHP<cd> h{cin(hp_re, hp_im, 0), cin(hp_re, hp_im, 1), cin(hp_re, hp_im, 2),
               cin(hp_re, hp_im, 3), cin(hp_re, hp_im, 4)};
  for (int64_t i = 0; i < n; ++i) {
    auto r = oracle::adam_fwd<cd>(cin(g_re, g_im, i), cin(m_re, m_im, i), cin(v_re, v_im, i), h, t);
    cout_(u_re, u_im, i, r.u);
    cout_(m1_re, m1_im, i, r.m1);
    cout_(v1_re, v1_im, i, r.v1);
  }
}

void oracle_rmsprop_fwd_cplx(int64_t n, const double* hp_re, const double* hp_im,
                             const double* g_re, const double* g_im, const double* v_re,
                             const double* v_im, double* u_re, double* u_im, double* v1_re,
                             double* v1_im) {
  RmsHP<cd> h{cin(hp_re, hp_im, 0), cin(hp_re, hp_im, 1), cin(hp_re, hp_im, 2)};
  for (int64_t i = 0; i < n; ++i) {
    auto r = oracle::rmsprop_fwd<cd>(cin(g_re, g_im, i), cin(v_re, v_im, i), h);
    cout_(u_re, u_im, i, r.u);
    cout_(v1_re, v1_im, i, r.v1);
  }
}

void oracle_sgd_fwd_cplx(int64_t n, const double* hp_re, const double* hp_im, int nesterov,
                         const double* g_re, const double* g_im, const double* b_re,
                         const double* b_im, double* u_re, double* u_im, double* b1_re,
                         double* b1_im) {
  SgdHP<cd> h{cin(hp_re, hp_im, 0), cin(hp_re, hp_im, 1), nesterov};
  for (int64_t i = 0; i < n; ++i) {
    auto r = oracle::sgd_fwd<cd>(cin(g_re, g_im, i), cin(b_re, b_im, i), h);
    cout_(u_re, u_im, i, r.u);
    cout_(b1_re, b1_im, i, r.b1);
  }
}

// Complex forward of the K-step map: theta_K per element (row a9 forward).
void oracle_sweep_forward_cplx(int kind, int64_t n, int64_t K, const double* hp_re,
                               const double* hp_im, int nesterov, const double* a,
                               const double* th0_re, const double* th0_im,
                               const double* phi_re, const double* phi_im,
                               double* thK_re, double* thK_im) {
  const int nhp = kind == 0 ? 5 : 3;
  cd hpc[5];
  for (int k = 0; k < nhp; ++k) hpc[k] = cin(hp_re, hp_im, k);
  for (int64_t i = 0; i < n; ++i) {
    cd th = cin(th0_re, th0_im, i), phi = cin(phi_re, phi_im, i);
    cd s1(0), s2(0);
    for (int64_t k = 0; k < K; ++k) {
      cd g = cd(a[i]) * (th - phi);
      cd u;
      if (kind == 0) {
        auto r = oracle::adam_fwd<cd>(g, s1, s2, AdamHP<cd>{hpc[0], hpc[1], hpc[2], hpc[3], hpc[4]}, k + 1);
        u = r.u; s1 = r.m1; s2 = r.v1;
      } else if (kind == 1) {
        auto r = oracle::rmsprop_fwd<cd>(g, s1, RmsHP<cd>{hpc[0], hpc[1], hpc[2]});
        u = r.u; s1 = r.v1;
      } else {
        auto r = oracle::sgd_fwd<cd>(g, s1, SgdHP<cd>{hpc[0], hpc[1], nesterov});
        u = r.u; s1 = r.b1;
      }
      th = th + u;
    }
    cout_(thK_re, thK_im, i, th);
  }
}

}  // extern "C"

// ---------------------------------------------- magnitude-twin entry points
// out[k*n + i]: per-element scales of the outputs in the order documented in
// oracle/__init__.py; hsum[k]: Sigma over elements of the hyper-term scales.
extern "C" {

void oracle_adam_mag(int64_t n, int64_t t, const double* hp, int bf, const float* g,
                     const void* m, const void* v, const float* du, const float* dm1,
                     const float* dv1, double* out, double* hsum, double* h_elem) {
  const AdamHP<double> h = adam_hp<double>(hp);
  long double hs[4] = {0, 0, 0, 0};
  for (int64_t i = 0; i < n; ++i) {
    auto r = oracle::adam_mag(f32_in(g, i), state_in(m, bf, i), state_in(v, bf, i), f32_in(du, i),
                              f32_in(dm1, i), f32_in(dv1, i), h, t);
    const double o[6] = {r.u, r.m1, r.v1, r.dg, r.dm, r.dv};
    for (int k = 0; k < 6; ++k) out[k * n + i] = o[k];
    for (int k = 0; k < 4; ++k) hs[k] += r.h[k];
    if (h_elem)
      for (int k = 0; k < 4; ++k) h_elem[k * n + i] = r.h[k];
  }
  for (int k = 0; k < 4; ++k) hsum[k] = (double)hs[k];
}

void oracle_rmsprop_mag(int64_t n, const double* hp, int bf, const float* g, const void* v,
                        const float* du, const float* dv1, double* out, double* hsum,
                        double* h_elem) {
  const RmsHP<double> h = rms_hp<double>(hp);
  long double hs[3] = {0, 0, 0};
  for (int64_t i = 0; i < n; ++i) {
    auto r = oracle::rmsprop_mag(f32_in(g, i), state_in(v, bf, i), f32_in(du, i), f32_in(dv1, i), h);
    const double o[4] = {r.u, r.v1, r.dg, r.dv};
    for (int k = 0; k < 4; ++k) out[k * n + i] = o[k];
    for (int k = 0; k < 3; ++k) hs[k] += r.h[k];
    if (h_elem)
      for (int k = 0; k < 3; ++k) h_elem[k * n + i] = r.h[k];
  }
  for (int k = 0; k < 3; ++k) hsum[k] = (double)hs[k];
}

void oracle_sgd_mag(int64_t n, const double* hp, int bf, const float* g, const void* b,
                    const float* du, const float* db1, double* out, double* hsum,
                    double* h_elem) {
  const SgdHP<double> h = sgd_hp<double>(hp);
  long double hs[2] = {0, 0};
  for (int64_t i = 0; i < n; ++i) {
    auto r = oracle::sgd_mag(f32_in(g, i), state_in(b, bf, i), f32_in(du, i), f32_in(db1, i), h);
    const double o[4] = {r.u, r.b1, r.dg, r.db};
    for (int k = 0; k < 4; ++k) out[k * n + i] = o[k];
    for (int k = 0; k < 2; ++k) hs[k] += r.h[k];
    if (h_elem)
      for (int k = 0; k < 2; ++k) h_elem[k * n + i] = r.h[k];
  }
  for (int k = 0; k < 2; ++k) hsum[k] = (double)hs[k];
}

}  // extern "C"

// ----------------------------------- optimizer variants (NEXT-1) entry points
// ext[3] = {weight_decay, decoupled, maximize}; lr_leaf (double[n_leaves]) or
// NULL: element i uses the learning rate of its leaf (offsets), else hp[0].
// Hyper-gradient slots: adam (lr, b1, b2, eps, wd), rmsprop (lr, alpha, eps,
// wd), sgd (lr, mu, wd); dhp_leaf[l*nh + k] are the same sums per leaf.
namespace {

template <class Fn>
void per_leaf_elements(int64_t n, int64_t n_leaves, const int64_t* off, Fn fn) {
  if (!off || n_leaves <= 0) {
    for (int64_t i = 0; i < n; ++i) fn(i, (int64_t)0);
    return;
  }
  for (int64_t l = 0; l < n_leaves; ++l)
    for (int64_t i = off[l]; i < off[l + 1]; ++i) fn(i, l);
}

template <class T>
oracle::ExHP<T> ex_hp(const double* ext) {
  return {T(ext[0]), ext[1] != 0.0 ? 1 : 0, ext[2] != 0.0 ? 1 : 0};
}

template <class T, int NH, class Elem>
void vjp_ex_loop(int64_t n, int64_t n_leaves, const int64_t* off, double* dhp, double* dhp_abs,
                 double* dhp_leaf, Elem elem) {
  long double s[NH] = {}, a[NH] = {};
  std::vector<long double> leaf((size_t)(n_leaves > 0 ? n_leaves : 1) * NH, 0.0L);
  per_leaf_elements(n, n_leaves, off, [&](int64_t i, int64_t l) {
    T h[NH];
    elem(i, l, h);
    for (int k = 0; k < NH; ++k) {
      long double x = (long double)h[k];
      s[k] += x;
      a[k] += x < 0 ? -x : x;
      leaf[(size_t)l * NH + k] += x;
    }
  });
  for (int k = 0; k < NH; ++k) {
    if (dhp) dhp[k] = (double)s[k];
    if (dhp_abs) dhp_abs[k] = (double)a[k];
  }
  if (dhp_leaf && off)
    for (int64_t l = 0; l < n_leaves; ++l)
      for (int k = 0; k < NH; ++k) dhp_leaf[l * NH + k] = (double)leaf[(size_t)l * NH + k];
}

template <class T>
void adam_fwd_ex_arr(int64_t n, int64_t t, const double* hp, const double* ext,
                     const double* lr_leaf, int64_t nl, const int64_t* off, int bf, const float* g,
                     const void* m, const void* v, const float* th, double* u, double* m1,
                     double* v1) {
  const oracle::ExHP<T> x = ex_hp<T>(ext);
  per_leaf_elements(n, nl, off, [&](int64_t i, int64_t l) {
    AdamHP<T> h = adam_hp<T>(hp);
    if (lr_leaf) h.lr = T(lr_leaf[l]);
    auto r = oracle::adam_fwd_ex<T>(T(f32_in(g, i)), T(state_in(m, bf, i)), T(state_in(v, bf, i)),
                                    T(f32_in(th, i)), h, x, t);
    put(u, i, (double)r.u);
    put(m1, i, (double)r.m1);
    put(v1, i, (double)r.v1);
  });
}

template <class T>
void adam_vjp_ex_arr(int64_t n, int64_t t, const double* hp, const double* ext,
                     const double* lr_leaf, int64_t nl, const int64_t* off, int bf, const float* g,
                     const void* m, const void* v, const float* th, const float* du,
                     const float* dm1, const float* dv1, double* dg, double* dm, double* dv,
                     double* dth, double* dhp, double* dhp_abs, double* dhp_leaf) {
  const oracle::ExHP<T> x = ex_hp<T>(ext);
  vjp_ex_loop<T, 5>(n, nl, off, dhp, dhp_abs, dhp_leaf, [&](int64_t i, int64_t l, T* h) {
    AdamHP<T> hh = adam_hp<T>(hp);
    if (lr_leaf) hh.lr = T(lr_leaf[l]);
    auto r = oracle::adam_vjp_ex<T>(T(f32_in(g, i)), T(state_in(m, bf, i)), T(state_in(v, bf, i)),
                                    T(f32_in(th, i)), T(f32_in(du, i)), T(f32_in(dm1, i)),
                                    T(f32_in(dv1, i)), hh, x, t);
    put(dg, i, (double)r.dg);
    put(dm, i, (double)r.dm);
    put(dv, i, (double)r.dv);
    put(dth, i, (double)r.dtheta);
    h[0] = r.dlr; h[1] = r.db1; h[2] = r.db2; h[3] = r.deps; h[4] = r.dwd;
  });
}

template <class T>
void rms_fwd_ex_arr(int64_t n, const double* hp, const double* ext, const double* lr_leaf,
                    int64_t nl, const int64_t* off, int bf, const float* g, const void* v,
                    const float* th, double* u, double* v1) {
  const oracle::ExHP<T> x = ex_hp<T>(ext);
  per_leaf_elements(n, nl, off, [&](int64_t i, int64_t l) {
    RmsHP<T> h = rms_hp<T>(hp);
    if (lr_leaf) h.lr = T(lr_leaf[l]);
    auto r = oracle::rmsprop_fwd_ex<T>(T(f32_in(g, i)), T(state_in(v, bf, i)), T(f32_in(th, i)),
                                       h, x);
    put(u, i, (double)r.u);
    put(v1, i, (double)r.v1);
  });
}

template <class T>
void rms_vjp_ex_arr(int64_t n, const double* hp, const double* ext, const double* lr_leaf,
                    int64_t nl, const int64_t* off, int bf, const float* g, const void* v,
                    const float* th, const float* du, const float* dv1, double* dg, double* dv,
                    double* dth, double* dhp, double* dhp_abs, double* dhp_leaf) {
  const oracle::ExHP<T> x = ex_hp<T>(ext);
  vjp_ex_loop<T, 4>(n, nl, off, dhp, dhp_abs, dhp_leaf, [&](int64_t i, int64_t l, T* h) {
    RmsHP<T> hh = rms_hp<T>(hp);
    if (lr_leaf) hh.lr = T(lr_leaf[l]);
    auto r = oracle::rmsprop_vjp_ex<T>(T(f32_in(g, i)), T(state_in(v, bf, i)), T(f32_in(th, i)),
                                       T(f32_in(du, i)), T(f32_in(dv1, i)), hh, x);
    put(dg, i, (double)r.dg);
    put(dv, i, (double)r.dv);
    put(dth, i, (double)r.dtheta);
    h[0] = r.dlr; h[1] = r.dalpha; h[2] = r.deps; h[3] = r.dwd;
  });
}

template <class T>
void sgd_fwd_ex_arr(int64_t n, const double* hp, const double* ext, const double* lr_leaf,
                    int64_t nl, const int64_t* off, int bf, const float* g, const void* b,
                    const float* th, double* u, double* b1) {
  const oracle::ExHP<T> x = ex_hp<T>(ext);
  per_leaf_elements(n, nl, off, [&](int64_t i, int64_t l) {
    SgdHP<T> h = sgd_hp<T>(hp);
    if (lr_leaf) h.lr = T(lr_leaf[l]);
    auto r = oracle::sgd_fwd_ex<T>(T(f32_in(g, i)), T(state_in(b, bf, i)), T(f32_in(th, i)), h, x);
    put(u, i, (double)r.u);
    put(b1, i, (double)r.b1);
  });
}

template <class T>
void sgd_vjp_ex_arr(int64_t n, const double* hp, const double* ext, const double* lr_leaf,
                    int64_t nl, const int64_t* off, int bf, const float* g, const void* b,
                    const float* th, const float* du, const float* db1, double* dg, double* db,
                    double* dth, double* dhp, double* dhp_abs, double* dhp_leaf) {
  const oracle::ExHP<T> x = ex_hp<T>(ext);
  vjp_ex_loop<T, 3>(n, nl, off, dhp, dhp_abs, dhp_leaf, [&](int64_t i, int64_t l, T* h) {
    SgdHP<T> hh = sgd_hp<T>(hp);
    if (lr_leaf) hh.lr = T(lr_leaf[l]);
    auto r = oracle::sgd_vjp_ex<T>(T(f32_in(g, i)), T(state_in(b, bf, i)), T(f32_in(th, i)),
                                   T(f32_in(du, i)), T(f32_in(db1, i)), hh, x);
    put(dg, i, (double)r.dg);
    put(db, i, (double)r.db);
    put(dth, i, (double)r.dtheta);
    h[0] = r.dlr; h[1] = r.dmu; h[2] = r.dwd;
  });
}

}  // namespace

extern "C" {

void oracle_adam_fwd_ex(int64_t n, int64_t t, const double* hp, const double* ext,
                        const double* lr_leaf, int64_t nl, const int64_t* off, int bf, int prec,
                        const float* g, const void* m, const void* v, const float* th, double* u,
                        double* m1, double* v1) {
  if (prec) adam_fwd_ex_arr<long double>(n, t, hp, ext, lr_leaf, nl, off, bf, g, m, v, th, u, m1, v1);
  else adam_fwd_ex_arr<double>(n, t, hp, ext, lr_leaf, nl, off, bf, g, m, v, th, u, m1, v1);
}

void oracle_adam_vjp_ex(int64_t n, int64_t t, const double* hp, const double* ext,
                        const double* lr_leaf, int64_t nl, const int64_t* off, int bf, int prec,
                        const float* g, const void* m, const void* v, const float* th,
                        const float* du, const float* dm1, const float* dv1, double* dg,
                        double* dm, double* dv, double* dth, double* dhp, double* dhp_abs,
                        double* dhp_leaf) {
  if (prec)
    adam_vjp_ex_arr<long double>(n, t, hp, ext, lr_leaf, nl, off, bf, g, m, v, th, du, dm1, dv1,
                                 dg, dm, dv, dth, dhp, dhp_abs, dhp_leaf);
  else
    adam_vjp_ex_arr<double>(n, t, hp, ext, lr_leaf, nl, off, bf, g, m, v, th, du, dm1, dv1, dg,
                            dm, dv, dth, dhp, dhp_abs, dhp_leaf);
}

void oracle_rmsprop_fwd_ex(int64_t n, const double* hp, const double* ext, const double* lr_leaf,
                           int64_t nl, const int64_t* off, int bf, int prec, const float* g,
                           const void* v, const float* th, double* u, double* v1) {
  if (prec) rms_fwd_ex_arr<long double>(n, hp, ext, lr_leaf, nl, off, bf, g, v, th, u, v1);
  else rms_fwd_ex_arr<double>(n, hp, ext, lr_leaf, nl, off, bf, g, v, th, u, v1);
}

void oracle_rmsprop_vjp_ex(int64_t n, const double* hp, const double* ext, const double* lr_leaf,
                           int64_t nl, const int64_t* off, int bf, int prec, const float* g,
                           const void* v, const float* th, const float* du, const float* dv1,
                           double* dg, double* dv, double* dth, double* dhp, double* dhp_abs,
                           double* dhp_leaf) {
  if (prec)
    rms_vjp_ex_arr<long double>(n, hp, ext, lr_leaf, nl, off, bf, g, v, th, du, dv1, dg, dv, dth,
                                dhp, dhp_abs, dhp_leaf);
  else
    rms_vjp_ex_arr<double>(n, hp, ext, lr_leaf, nl, off, bf, g, v, th, du, dv1, dg, dv, dth, dhp,
                           dhp_abs, dhp_leaf);
}

void oracle_sgd_fwd_ex(int64_t n, const double* hp, const double* ext, const double* lr_leaf,
                       int64_t nl, const int64_t* off, int bf, int prec, const float* g,
                       const void* b, const float* th, double* u, double* b1) {
  if (prec) sgd_fwd_ex_arr<long double>(n, hp, ext, lr_leaf, nl, off, bf, g, b, th, u, b1);
  else sgd_fwd_ex_arr<double>(n, hp, ext, lr_leaf, nl, off, bf, g, b, th, u, b1);
}

void oracle_sgd_vjp_ex(int64_t n, const double* hp, const double* ext, const double* lr_leaf,
                       int64_t nl, const int64_t* off, int bf, int prec, const float* g,
                       const void* b, const float* th, const float* du, const float* db1,
                       double* dg, double* db, double* dth, double* dhp, double* dhp_abs,
                       double* dhp_leaf) {
  if (prec)
    sgd_vjp_ex_arr<long double>(n, hp, ext, lr_leaf, nl, off, bf, g, b, th, du, db1, dg, db, dth,
                                dhp, dhp_abs, dhp_leaf);
  else
    sgd_vjp_ex_arr<double>(n, hp, ext, lr_leaf, nl, off, bf, g, b, th, du, db1, dg, db, dth, dhp,
                           dhp_abs, dhp_leaf);
}

// complex forward of the variants (complex-step pins); per-ELEMENT lr
// (lr_re/lr_im of n) so that a per-leaf lr perturbation can be expressed.
void oracle_adam_fwd_ex_cplx(int64_t n, int64_t t, const double* hp_re, const double* hp_im,
                             double wd_re, double wd_im, int decoupled, int maximize,
                             const double* lr_re, const double* lr_im, const double* g_re,
                             const double* g_im, const double* m_re, const double* m_im,
                             const double* v_re, const double* v_im, const double* th_re,
                             const double* th_im, double* u_re, double* u_im, double* m1_re,
                             double* m1_im, double* v1_re, double* v1_im) {
  oracle::ExHP<cd> x{cd(wd_re, wd_im), decoupled, maximize};
  for (int64_t i = 0; i < n; ++i) {
    AdamHP<cd> h{cin(lr_re, lr_im, i), cin(hp_re, hp_im, 1), cin(hp_re, hp_im, 2),
                 cin(hp_re, hp_im, 3), cin(hp_re, hp_im, 4)};
    auto r = oracle::adam_fwd_ex<cd>(cin(g_re, g_im, i), cin(m_re, m_im, i), cin(v_re, v_im, i),
                                     cin(th_re, th_im, i), h, x, t);
    cout_(u_re, u_im, i, r.u);
    cout_(m1_re, m1_im, i, r.m1);
    cout_(v1_re, v1_im, i, r.v1);
  }
}

void oracle_rmsprop_fwd_ex_cplx(int64_t n, const double* hp_re, const double* hp_im, double wd_re,
                                double wd_im, int maximize, const double* lr_re,
                                const double* lr_im, const double* g_re, const double* g_im,
                                const double* v_re, const double* v_im, const double* th_re,
                                const double* th_im, double* u_re, double* u_im, double* v1_re,
                                double* v1_im) {
  oracle::ExHP<cd> x{cd(wd_re, wd_im), 0, maximize};
  for (int64_t i = 0; i < n; ++i) {
    RmsHP<cd> h{cin(lr_re, lr_im, i), cin(hp_re, hp_im, 1), cin(hp_re, hp_im, 2)};
    auto r = oracle::rmsprop_fwd_ex<cd>(cin(g_re, g_im, i), cin(v_re, v_im, i),
                                        cin(th_re, th_im, i), h, x);
    cout_(u_re, u_im, i, r.u);
    cout_(v1_re, v1_im, i, r.v1);
  }
}

void oracle_sgd_fwd_ex_cplx(int64_t n, const double* hp_re, const double* hp_im, int nesterov,
                            double wd_re, double wd_im, int maximize, const double* lr_re,
                            const double* lr_im, const double* g_re, const double* g_im,
                            const double* b_re, const double* b_im, const double* th_re,
                            const double* th_im, double* u_re, double* u_im, double* b1_re,
                            double* b1_im) {
  oracle::ExHP<cd> x{cd(wd_re, wd_im), 0, maximize};
  for (int64_t i = 0; i < n; ++i) {
    SgdHP<cd> h{cin(lr_re, lr_im, i), cin(hp_re, hp_im, 1), nesterov};
    auto r = oracle::sgd_fwd_ex<cd>(cin(g_re, g_im, i), cin(b_re, b_im, i), cin(th_re, th_im, i),
                                    h, x);
    cout_(u_re, u_im, i, r.u);
    cout_(b1_re, b1_im, i, r.b1);
  }
}

}  // extern "C"

// ------------------------- RMSProp centred / momentum (NEXT-1) entry points
// hp[5] = {lr, alpha, eps, momentum, centered}; ext[3] as above (decoupled
// ignored); states v, a (gradient average), b (momentum buffer) may be NULL
// (zero). Hyper slots (lr, alpha, eps, momentum, wd).
namespace {

template <class T>
oracle::RmsCmHP<T> rms_cm_hp(const double* hp) {
  return {T(hp[0]), T(hp[1]), T(hp[2]), T(hp[3]), hp[4] != 0.0 ? 1 : 0};
}

template <class T>
void rms_cm_fwd_arr(int64_t n, const double* hp, const double* ext, const double* lr_leaf,
                    int64_t nl, const int64_t* off, int bf, const float* g, const void* v,
                    const void* a, const void* b, const float* th, double* u, double* v1,
                    double* a1, double* b1) {
  oracle::ExHP<T> x = ex_hp<T>(ext);
  x.decoupled = 0;
  per_leaf_elements(n, nl, off, [&](int64_t i, int64_t l) {
    oracle::RmsCmHP<T> h = rms_cm_hp<T>(hp);
    if (lr_leaf) h.lr = T(lr_leaf[l]);
    auto r = oracle::rmsprop_cm_fwd<T>(T(f32_in(g, i)), T(state_in(v, bf, i)),
                                       T(state_in(a, bf, i)), T(state_in(b, bf, i)),
                                       T(f32_in(th, i)), h, x);
    put(u, i, (double)r.u);
    put(v1, i, (double)r.v1);
    put(a1, i, (double)r.a1);
    put(b1, i, (double)r.b1);
  });
}

template <class T>
void rms_cm_vjp_arr(int64_t n, const double* hp, const double* ext, const double* lr_leaf,
                    int64_t nl, const int64_t* off, int bf, const float* g, const void* v,
                    const void* a, const void* b, const float* th, const float* du,
                    const float* dv1, const float* da1, const float* db1, double* dg, double* dv,
                    double* da, double* db, double* dth, double* dhp, double* dhp_abs,
                    double* dhp_leaf) {
  oracle::ExHP<T> x = ex_hp<T>(ext);
  x.decoupled = 0;
  vjp_ex_loop<T, 5>(n, nl, off, dhp, dhp_abs, dhp_leaf, [&](int64_t i, int64_t l, T* h) {
    oracle::RmsCmHP<T> hh = rms_cm_hp<T>(hp);
    if (lr_leaf) hh.lr = T(lr_leaf[l]);
    auto r = oracle::rmsprop_cm_vjp<T>(T(f32_in(g, i)), T(state_in(v, bf, i)),
                                       T(state_in(a, bf, i)), T(state_in(b, bf, i)),
                                       T(f32_in(th, i)), T(f32_in(du, i)), T(f32_in(dv1, i)),
                                       T(f32_in(da1, i)), T(f32_in(db1, i)), hh, x);
    put(dg, i, (double)r.dg);
    put(dv, i, (double)r.dv);
    put(da, i, (double)r.da);
    put(db, i, (double)r.db);
    put(dth, i, (double)r.dtheta);
    h[0] = r.dlr; h[1] = r.dalpha; h[2] = r.deps; h[3] = r.dmu; h[4] = r.dwd;
  });
}

}  // namespace

extern "C" {

void oracle_rmsprop_cm_fwd(int64_t n, const double* hp, const double* ext, const double* lr_leaf,
                           int64_t nl, const int64_t* off, int bf, int prec, const float* g,
                           const void* v, const void* a, const void* b, const float* th,
                           double* u, double* v1, double* a1, double* b1) {
  if (prec) rms_cm_fwd_arr<long double>(n, hp, ext, lr_leaf, nl, off, bf, g, v, a, b, th, u, v1, a1, b1);
  else rms_cm_fwd_arr<double>(n, hp, ext, lr_leaf, nl, off, bf, g, v, a, b, th, u, v1, a1, b1);
}

void oracle_rmsprop_cm_vjp(int64_t n, const double* hp, const double* ext, const double* lr_leaf,
                           int64_t nl, const int64_t* off, int bf, int prec, const float* g,
                           const void* v, const void* a, const void* b, const float* th,
                           const float* du, const float* dv1, const float* da1, const float* db1,
                           double* dg, double* dv, double* da, double* db, double* dth,
                           double* dhp, double* dhp_abs, double* dhp_leaf) {
  if (prec)
    rms_cm_vjp_arr<long double>(n, hp, ext, lr_leaf, nl, off, bf, g, v, a, b, th, du, dv1, da1,
                                db1, dg, dv, da, db, dth, dhp, dhp_abs, dhp_leaf);
  else
    rms_cm_vjp_arr<double>(n, hp, ext, lr_leaf, nl, off, bf, g, v, a, b, th, du, dv1, da1, db1,
                           dg, dv, da, db, dth, dhp, dhp_abs, dhp_leaf);
}

// Magnitude twins: out[k*n + i] for k = u, v1, a1, b1, dg, dv, da, db, dtheta;
// hsum[5] = Sigma of the hyper twins (element lr from lr_leaf when given).
void oracle_rmsprop_cm_mag(int64_t n, const double* hp, const double* ext,
                           const double* lr_leaf, int64_t nl, const int64_t* off, int bf,
                           const float* g, const void* v, const void* a, const void* b,
                           const float* th, const float* du, const float* dv1, const float* da1,
                           const float* db1, double* out, double* hsum, double* h_elem) {
  oracle::ExHP<double> x = ex_hp<double>(ext);
  x.decoupled = 0;
  long double hs[5] = {0, 0, 0, 0, 0};
  per_leaf_elements(n, nl, off, [&](int64_t i, int64_t l) {
    oracle::RmsCmHP<double> h = rms_cm_hp<double>(hp);
    if (lr_leaf) h.lr = lr_leaf[l];
    auto r = oracle::rmsprop_cm_mag(f32_in(g, i), state_in(v, bf, i), state_in(a, bf, i),
                                    state_in(b, bf, i), f32_in(th, i), f32_in(du, i),
                                    f32_in(dv1, i), f32_in(da1, i), f32_in(db1, i), h, x);
    const double o[9] = {r.u, r.v1, r.a1, r.b1, r.dg, r.dv, r.da, r.db, r.dtheta};
    for (int k = 0; k < 9; ++k) out[k * n + i] = o[k];
    for (int k = 0; k < 5; ++k) hs[k] += r.h[k];
    if (h_elem)
      for (int k = 0; k < 5; ++k) h_elem[k * n + i] = r.h[k];
  });
  for (int k = 0; k < 5; ++k) hsum[k] = (double)hs[k];
}

// Magnitude twins of the *_ex variants (oracle::ex_mag): kind 0 adam
// (hp = lr, b1, b2, eps, eps_root), 1 rmsprop (lr, alpha, eps), 2 sgd (lr,
// mu, nesterov). out[k*n + i] for k = u, s0', s1', dg, ds0, ds1, dtheta;
// hsum / h_elem[k*n + i] for the hyper slots (adam: lr, b1, b2, eps, wd;
// rmsprop: lr, alpha, eps, wd; sgd: lr, mu, wd).
void oracle_ex_mag(int kind, int64_t n, int64_t t, const double* hp, const double* ext,
                   const double* lr_leaf, int64_t nl, const int64_t* off, int bf, const float* g,
                   const void* s0, const void* s1, const float* th, const float* du,
                   const float* ds0, const float* ds1, double* out, double* hsum,
                   double* h_elem) {
  const oracle::ExHP<double> x = ex_hp<double>(ext);
  const int nh = kind == 0 ? 5 : kind == 1 ? 4 : 3;
  long double hs[5] = {0, 0, 0, 0, 0};
  per_leaf_elements(n, nl, off, [&](int64_t i, int64_t l) {
    double hh[5];
    for (int k = 0; k < 5; ++k) hh[k] = k < (kind == 0 ? 5 : 3) ? hp[k] : 0.0;
    if (lr_leaf) hh[0] = lr_leaf[l];
    auto r = oracle::ex_mag(kind, f32_in(g, i), state_in(s0, bf, i), state_in(s1, bf, i),
                            f32_in(th, i), f32_in(du, i), f32_in(ds0, i), f32_in(ds1, i), hh, x,
                            t);
    const double o[7] = {r.u, r.s0, r.s1, r.dg, r.ds0, r.ds1, r.dtheta};
    for (int k = 0; k < 7; ++k) out[k * n + i] = o[k];
    for (int k = 0; k < nh; ++k) {
      hs[k] += r.h[k];
      if (h_elem) h_elem[k * n + i] = r.h[k];
    }
  });
  for (int k = 0; k < nh; ++k) hsum[k] = (double)hs[k];
}

// Complex forward (complex-step pins); per-ELEMENT lr; hp_re/hp_im[4] =
// (lr unused, alpha, eps, momentum).
void oracle_rmsprop_cm_fwd_cplx(int64_t n, const double* hp_re, const double* hp_im,
                                int centered, double wd_re, double wd_im, int maximize,
                                const double* lr_re, const double* lr_im, const double* g_re,
                                const double* g_im, const double* v_re, const double* v_im,
                                const double* a_re, const double* a_im, const double* b_re,
                                const double* b_im, const double* th_re, const double* th_im,
                                double* u_re, double* u_im, double* v1_re, double* v1_im,
                                double* a1_re, double* a1_im, double* b1_re, double* b1_im) {
  oracle::ExHP<cd> x{cd(wd_re, wd_im), 0, maximize};
  for (int64_t i = 0; i < n; ++i) {
    oracle::RmsCmHP<cd> h{cin(lr_re, lr_im, i), cin(hp_re, hp_im, 1), cin(hp_re, hp_im, 2),
                          cin(hp_re, hp_im, 3), centered};
    auto r = oracle::rmsprop_cm_fwd<cd>(cin(g_re, g_im, i), cin(v_re, v_im, i),
                                        cin(a_re, a_im, i), cin(b_re, b_im, i),
                                        cin(th_re, th_im, i), h, x);
    cout_(u_re, u_im, i, r.u);
    cout_(v1_re, v1_im, i, r.v1);
    cout_(a1_re, a1_im, i, r.a1);
    cout_(b1_re, b1_im, i, r.b1);
  }
}

}  // extern "C"

// ------------------------------------------------ zero-order ES (NEXT-3)
extern "C" {

// z[i][j] for i < n_samples, j < numel (the noise itself, for tests).
void oracle_es_noise(int64_t numel, int64_t n_samples, uint64_t seed, double* z) {
  for (int64_t i = 0; i < n_samples; ++i)
    for (int64_t j = 0; j < numel; ++j) z[i * numel + j] = oracle::es_normal(seed, i, j);
}

// Perturbed points, row r of out: theta + sigma z_i (naive: r = i;
// antithetic: r = 2i is +, r = 2i+1 is -).
void oracle_es_perturb(int64_t numel, int64_t n_samples, int antithetic, double sigma,
                       uint64_t seed, const float* theta, double* out) {
  const int reps = antithetic ? 2 : 1;
  for (int64_t i = 0; i < n_samples; ++i)
    for (int64_t j = 0; j < numel; ++j) {
      const double z = oracle::es_normal(seed, i, j);
      out[(i * reps) * numel + j] = (double)theta[j] + sigma * z;
      if (antithetic) out[(i * reps + 1) * numel + j] = (double)theta[j] - sigma * z;
    }
}

// Gradient estimate from the f values of the perturbed points (same row
// order as oracle_es_perturb). g_abs (optional): sum over i of |term|.
void oracle_es_grad(int64_t numel, int64_t n_samples, int antithetic, double sigma,
                    uint64_t seed, const double* f, double* g, double* g_abs) {
  const double scale = antithetic ? 1.0 / (2.0 * n_samples * sigma) : 1.0 / (n_samples * sigma);
  for (int64_t j = 0; j < numel; ++j) {
    long double s = 0.0L, a = 0.0L;
    for (int64_t i = 0; i < n_samples; ++i) {
      const double w = antithetic ? f[2 * i] - f[2 * i + 1] : f[i];
      const long double term = (long double)w * oracle::es_normal(seed, i, j);
      s += term;
      a += term < 0 ? -term : term;
    }
    g[j] = (double)(s * scale);
    if (g_abs) g_abs[j] = (double)(a * (scale < 0 ? -scale : scale));
  }
}

}  // extern "C"

// ---------------------------------------- implicit gradients (NEXT-4)
// PAPER.md §2.2 "Implicit Gradient (IG)": the best-response
// derivative comes from the implicit function theorem, which needs linear
// solves with dF/dtheta; TorchOpt offers conjugate gradient (iMAML) and
// Neumann series solvers. Plain textbook forms on explicit data:
//   CG: r0 = b - A x0, p0 = r0; alpha = r.r / p.Ap; x += alpha p;
//       r -= alpha Ap; beta = r'.r' / r.r; p = r' + beta p
//   Neumann: x = alpha sum_{k=0}^{K} (I - alpha A)^k b
extern "C" {

// One CG iteration on given vectors (fp32 inputs as the GPU holds them):
// outputs x', r', p' and scalars s = {pAp, alpha, rr_new, beta}.
void oracle_cg_iter(int64_t n, const float* x, const float* r, const float* p, const float* Ap,
                    double rr, double* x1, double* r1, double* p1, double* s) {
  long double pap = 0.0L;
  for (int64_t i = 0; i < n; ++i) pap += (long double)p[i] * (long double)Ap[i];
  const double alpha = pap == 0.0L ? 0.0 : rr / (double)pap;
  long double rrn = 0.0L;
  for (int64_t i = 0; i < n; ++i) {
    x1[i] = (double)x[i] + alpha * (double)p[i];
    r1[i] = (double)r[i] - alpha * (double)Ap[i];
    rrn += (long double)r1[i] * r1[i];
  }
  const double beta = rr == 0.0 ? 0.0 : (double)rrn / rr;
  for (int64_t i = 0; i < n; ++i) p1[i] = r1[i] + beta * (double)p[i];
  s[0] = (double)pap;
  s[1] = alpha;
  s[2] = (double)rrn;
  s[3] = beta;
}

// CG on a dense row-major SPD matrix, `iters` iterations from x0 = 0.
void oracle_cg_dense(int64_t n, const double* A, const double* b, int64_t iters, double* x) {
  std::vector<double> r(b, b + n), p(b, b + n), Ap(n);
  for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
  double rr = 0.0;
  for (int64_t i = 0; i < n; ++i) rr += r[i] * r[i];
  for (int64_t it = 0; it < iters && rr > 0.0; ++it) {
    for (int64_t i = 0; i < n; ++i) {
      double s = 0.0;
      for (int64_t j = 0; j < n; ++j) s += A[i * n + j] * p[j];
      Ap[i] = s;
    }
    double pap = 0.0;
    for (int64_t i = 0; i < n; ++i) pap += p[i] * Ap[i];
    const double alpha = rr / pap;
    double rrn = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * Ap[i];
      rrn += r[i] * r[i];
    }
    const double beta = rrn / rr;
    for (int64_t i = 0; i < n; ++i) p[i] = r[i] + beta * p[i];
    rr = rrn;
  }
}

// Truncated Neumann series x = alpha sum_{k=0}^{K} (I - alpha A)^k b (dense).
void oracle_neumann_dense(int64_t n, const double* A, const double* b, int64_t K, double alpha,
                          double* x) {
  std::vector<double> v(n), t(n);
  for (int64_t i = 0; i < n; ++i) {
    v[i] = alpha * b[i];  // alpha (I - alpha A)^0 b
    x[i] = v[i];
  }
  for (int64_t k = 1; k <= K; ++k) {
    for (int64_t i = 0; i < n; ++i) {
      double s = 0.0;
      for (int64_t j = 0; j < n; ++j) s += A[i * n + j] * v[j];
      t[i] = v[i] - alpha * s;
    }
    for (int64_t i = 0; i < n; ++i) {
      v[i] = t[i];
      x[i] += v[i];
    }
  }
}

}  // extern "C"
