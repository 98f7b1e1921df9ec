/* include/diffopt.h -- C ABI of the B200 fused differentiable optimizer step.
 *
 * What the library computes (PAPER.md = P:, SPEC.md = S:, SURVEY.md = SV):
 *   The paper's "CPU/GPU-accelerated optimizers" take "the optimizer as a
 *   whole instead of separating it into several basic operators", with the
 *   forward and backward written by hand, "symbolic reduction" and explicit
 *   0/0 cancellation (§2.3; contribution (2)(i), P:36 names SGD,
 *   RMSProp and Adam). This library is that operator for sm_100a: one fused
 *   pass over HBM for the update (forward) and one for its vector-Jacobian
 *   product (backward) with respect to the gradient, the optimizer state and
 *   the hyper-parameters. The update formulas are the standard ones quoted in
 *   S:188 (Adam), S:196-204 (SGD-momentum), S:206 (RMSProp); every reading
 *   of a point the paper leaves open is listed in DESIGN.md ("Readings").
 *
 * Data layout (SV §8(b), P:87 / P:248 tensor trees):
 *   A tensor tree is flattened once on the host into ONE contiguous buffer
 *   per role (gradient, each state slot, update, each cotangent). Leaves are
 *   contiguous segments [offsets[l], offsets[l+1]) in depth-first leaf order
 *   (S:123). All element arrays are indexed by the same flat index.
 *   fp32 arrays are `float`; state arrays (mu, nu, momentum buffer) are
 *   `float` when state_dtype == OPT_F32 and bf16 (`uint16_t` bit patterns)
 *   when state_dtype == OPT_BF16 (reading Z9: only persistent state is
 *   bf16; gradients, updates and all cotangents stay fp32).
 *
 * Conventions shared by every entry point:
 *   - All array pointers are DEVICE pointers (cudaMalloc'd, or mapped host
 *     memory) and must be 16-byte aligned (else OPT_EALIGN).
 *   - A NULL state input means the zero state (opt.init); a NULL
 *     cotangent means a zero cotangent (bitwise identical result); a NULL
 *     output is not written.
 *   - Exact aliasing of an output with the input it replaces is allowed
 *     (mu_out == mu, nu_out == nu, updates == g, d_g == d_updates,
 *     d_mu == d_mu_out, d_nu == d_nu_out, params_out == params); every element
 *     is read before it is written. Any other overlap is undefined.
 *   - The caller owns every buffer. The library allocates nothing, keeps no
 *     per-call state, never synchronises the device and enqueues all work on
 *     `stream` (a cudaStream_t; NULL = legacy default stream).
 *   - Host-side validation runs before anything is enqueued; on error nothing
 *     is launched and the thread-local message is set (opt_last_error).
 *     Device-side NaN/Inf inputs propagate; they are not checked.
 *   - numel == 0 is valid: nothing is launched except zeroing d_hp/d_hp_leaf
 *     (cudaMemsetAsync on `stream`).
 *   - Hyper-gradient outputs d_hp / d_hp_leaf are device double arrays that
 *     are WRITTEN (not accumulated). Their reduction order is fixed, so they
 *     are bitwise reproducible run to run on one device (reading Z12).
 *   - Thread-safe and re-entrant; concurrent calls must not share a
 *     workspace.
 */
#ifndef DIFFOPT_H
#define DIFFOPT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DIFFOPT_ABI_VERSION 6

typedef enum {
  OPT_OK = 0,
  OPT_EINVAL = 1,      /* invalid argument (hyper-parameter range, sizes, offsets) */
  OPT_EALIGN = 2,      /* an array pointer is not 16-byte aligned */
  OPT_ECUDA = 3,       /* a CUDA call or launch failed (message in opt_last_error) */
  OPT_EWORKSPACE = 4   /* workspace missing or smaller than opt_workspace_bytes() */
} opt_status;

typedef enum { OPT_F32 = 0, OPT_BF16 = 1 } opt_state_dtype;

/* Arithmetic precision inside the kernel. Storage is unchanged (fp32 arrays,
 * state per opt_state_dtype); only the per-element arithmetic differs.
 * OPT_COMPUTE_DEFAULT picks the library default. */
typedef enum { OPT_COMPUTE_DEFAULT = 0, OPT_COMPUTE_F32 = 1, OPT_COMPUTE_F64 = 2 } opt_compute;

/* The flattened tree (SV §8(a) row a1). offsets has n_leaves + 1 int64
 * entries, offsets[0] = 0, non-decreasing, offsets[n_leaves] = numel.
 * h_offsets (host) is always required when n_leaves > 0; d_offsets (device
 * copy of the same values) is required only when per-leaf outputs are
 * requested. n_leaves == 0 means "one leaf of numel elements". Caller-owned. */
typedef struct {
  int64_t numel;
  int64_t n_leaves;
  const int64_t* h_offsets;
  const int64_t* d_offsets;
} opt_tree;

/* Adam: m' = b1 m + (1-b1) g ; v' = b2 v + (1-b2) g^2 ;
 *   u = -lr (m'/(1-b1^t)) / (sqrt(v'/(1-b2^t) + eps_root) + eps).
 * Valid: lr finite, 0 <= b1 < 1, 0 <= b2 < 1, eps >= 0, eps_root >= 0. */
typedef struct { double lr, b1, b2, eps, eps_root; } opt_adam_hp;
/* RMSProp: v' = alpha v + (1-alpha) g^2 ; u = -lr g/(sqrt(v') + eps).
 * Valid: lr finite, 0 <= alpha < 1, eps >= 0. */
typedef struct { double lr, alpha, eps; } opt_rmsprop_hp;
/* SGD: b' = momentum b + g ; u = -lr b' (nesterov: -lr (g + momentum b')).
 * Valid: lr finite, 0 <= momentum < 1. */
typedef struct { double lr, momentum; int nesterov; } opt_sgd_hp;

/* Bytes of device workspace a backward call needs (per_leaf != 0 when
 * d_hp_leaf will be requested). The workspace must be zero-filled once
 * when allocated; every call leaves it zero-filled again. Returns 0 and
 * sets opt_last_error on an invalid tree. */
size_t opt_workspace_bytes(const opt_tree* tree, int per_leaf);

/* ------------------------------------------------------------------ Adam
 * Forward (SV §8(a) row a3). Reads g, mu, nu (+ params); writes updates,
 * mu_out, nu_out and, when params and params_out are both non-NULL,
 * params_out = params + updates (apply_updates fused; updates may then
 * be NULL). step = t >= 1 (reading Z3).
 * Returns OPT_OK / OPT_EINVAL / OPT_EALIGN / OPT_ECUDA. */
int opt_adam_fwd(const opt_tree* tree, int64_t step, const opt_adam_hp* hp,
                 int state_dtype, int compute,
                 const float* g, const void* mu, const void* nu,
                 float* updates, void* mu_out, void* nu_out,
                 const float* params, float* params_out, void* stream);

/* Backward (VJP; SV §8(a) rows a4, a5). Given the forward's inputs g, mu, nu
 * and the cotangents d_updates, d_mu_out, d_nu_out of its outputs, writes
 * d_g, d_mu, d_nu (fp32) and, if non-NULL, d_hp[4] = (lr, b1, b2, eps)
 * hyper-gradients summed over all elements, and d_hp_leaf[n_leaves][4] the
 * same sums per leaf (needs tree->d_offsets; any leaf count). eps_root
 * is not differentiated. workspace: see opt_workspace_bytes. */
int opt_adam_bwd(const opt_tree* tree, int64_t step, const opt_adam_hp* hp,
                 int state_dtype, int compute,
                 const float* g, const void* mu, const void* nu,
                 const float* d_updates, const float* d_mu_out, const float* d_nu_out,
                 float* d_g, float* d_mu, float* d_nu,
                 double* d_hp, double* d_hp_leaf,
                 void* workspace, size_t workspace_bytes, void* stream);

/* --------------------------------------------------------------- RMSProp
 * As Adam with one state array nu; d_hp[3] = (lr, alpha, eps). */
int opt_rmsprop_fwd(const opt_tree* tree, const opt_rmsprop_hp* hp,
                    int state_dtype, int compute,
                    const float* g, const void* nu,
                    float* updates, void* nu_out,
                    const float* params, float* params_out, void* stream);

int opt_rmsprop_bwd(const opt_tree* tree, const opt_rmsprop_hp* hp,
                    int state_dtype, int compute,
                    const float* g, const void* nu,
                    const float* d_updates, const float* d_nu_out,
                    float* d_g, float* d_nu,
                    double* d_hp, double* d_hp_leaf,
                    void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------- SGD
 * State = momentum buffer (may be NULL on input = zero buffer; mom_out may
 * be NULL when momentum == 0). d_hp[2] = (lr, momentum). */
int opt_sgd_fwd(const opt_tree* tree, const opt_sgd_hp* hp,
                int state_dtype, int compute,
                const float* g, const void* mom,
                float* updates, void* mom_out,
                const float* params, float* params_out, void* stream);

int opt_sgd_bwd(const opt_tree* tree, const opt_sgd_hp* hp,
                int state_dtype, int compute,
                const float* g, const void* mom,
                const float* d_updates, const float* d_mom_out,
                float* d_g, float* d_mom,
                double* d_hp, double* d_hp_leaf,
                void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------- optimizer variants (SV §8(f) NEXT-1)
 * The paper's optimizers are the plain ones; these variants follow
 * torch.optim semantics (reading N1) and make hyper-parameters
 * beyond lr/betas/eps meta-learnable (MGRL-style meta-gradients):
 *   maximize      : the step ascends: g is replaced by -g first;
 *   weight_decay  : L2 (all three): g~ = (maximize ? -g : g) + wd * theta,
 *                   or, Adam with decoupled = 1 (AdamW): u += -lr * wd * theta;
 *   lr_leaf       : device float[n_leaves]; leaf l uses lr_leaf[l] instead of
 *                   hp->lr (per-leaf learnable learning rates). Needs
 *                   tree->d_offsets (any leaf count); the per-leaf lr
 *                   gradients are slot 0 of d_hp_leaf.
 * theta = params (required when weight_decay != 0). The *_ex forward writes
 * params_out = params + updates when both are non-NULL. The *_ex backward
 * writes d_params = the cotangent of params THROUGH THE UPDATE ONLY (the
 * weight-decay path); a caller that fused apply_updates adds d_updates for
 * the identity. Hyper-gradient slots gain weight_decay as the last slot:
 * Adam (lr, b1, b2, eps, wd), RMSProp (lr, alpha, eps, wd), SGD (lr, mu, wd). */
typedef struct {
  double weight_decay;   /* >= 0 */
  int decoupled;         /* Adam only: 1 = AdamW decoupled decay */
  int maximize;          /* 1 = gradient ascent */
  const float* lr_leaf;  /* device [n_leaves] or NULL; 16-byte aligned */
} opt_ext;

int opt_adam_fwd_ex(const opt_tree* tree, int64_t step, const opt_adam_hp* hp, const opt_ext* ext,
                    int state_dtype, int compute, const float* g, const void* mu, const void* nu,
                    const float* params, float* updates, void* mu_out, void* nu_out,
                    float* params_out, void* stream);
int opt_adam_bwd_ex(const opt_tree* tree, int64_t step, const opt_adam_hp* hp, const opt_ext* ext,
                    int state_dtype, int compute, const float* g, const void* mu, const void* nu,
                    const float* params, const float* d_updates, const float* d_mu_out,
                    const float* d_nu_out, float* d_g, float* d_mu, float* d_nu, float* d_params,
                    double* d_hp, double* d_hp_leaf, void* workspace, size_t workspace_bytes,
                    void* stream);
int opt_rmsprop_fwd_ex(const opt_tree* tree, const opt_rmsprop_hp* hp, const opt_ext* ext,
                       int state_dtype, int compute, const float* g, const void* nu,
                       const float* params, float* updates, void* nu_out, float* params_out,
                       void* stream);
int opt_rmsprop_bwd_ex(const opt_tree* tree, const opt_rmsprop_hp* hp, const opt_ext* ext,
                       int state_dtype, int compute, const float* g, const void* nu,
                       const float* params, const float* d_updates, const float* d_nu_out,
                       float* d_g, float* d_nu, float* d_params, double* d_hp, double* d_hp_leaf,
                       void* workspace, size_t workspace_bytes, void* stream);
/* Centred and/or momentum RMSProp (SURVEY §8(f) NEXT-1 "centered and
 * momentum RMSProp"; torch.optim.RMSprop semantics, reading N4):
 *   g~ = (maximize ? -g : g) + weight_decay * params   (ext; decoupled ignored)
 *   v' = alpha v + (1-alpha) g~^2
 *   centered: a' = alpha a + (1-alpha) g~, q = v' - a'^2   (else q = v')
 *   d = sqrt(q) + eps  (sqrt(q <= 0) := 0),  w = g~/d  (0 at d = 0)
 *   b' = momentum b + w,  u = -lr b'   (momentum = 0: u = -lr g~/d)
 * State: nu (square average), gavg (gradient average; used only when
 * centered), buf (momentum buffer); each may be NULL on input (zero state)
 * and NULL on output (not written). Valid: lr finite, 0 <= alpha < 1,
 * eps >= 0, 0 <= momentum < 1. Per-leaf lr via ext->lr_leaf. */
typedef struct { double lr, alpha, eps, momentum; int centered; } opt_rmsprop_cm_hp;
int opt_rmsprop_cm_fwd(const opt_tree* tree, const opt_rmsprop_cm_hp* hp, const opt_ext* ext,
                       int state_dtype, int compute, const float* g, const void* nu,
                       const void* gavg, const void* buf, const float* params, float* updates,
                       void* nu_out, void* gavg_out, void* buf_out, float* params_out,
                       void* stream);
/* Backward: cotangents of (updates, nu_out, gavg_out, buf_out) in; d_g,
 * d_nu, d_gavg, d_buf and d_params (through the update only; add d_updates
 * for a fused apply) out; d_hp[5] = (lr, alpha, eps, momentum,
 * weight_decay) sums, d_hp_leaf[n_leaves][5] per leaf. */
int opt_rmsprop_cm_bwd(const opt_tree* tree, const opt_rmsprop_cm_hp* hp, const opt_ext* ext,
                       int state_dtype, int compute, const float* g, const void* nu,
                       const void* gavg, const void* buf, const float* params,
                       const float* d_updates, const float* d_nu_out, const float* d_gavg_out,
                       const float* d_buf_out, float* d_g, float* d_nu, float* d_gavg,
                       float* d_buf, float* d_params, double* d_hp, double* d_hp_leaf,
                       void* workspace, size_t workspace_bytes, void* stream);
int opt_sgd_fwd_ex(const opt_tree* tree, const opt_sgd_hp* hp, const opt_ext* ext,
                   int state_dtype, int compute, const float* g, const void* mom,
                   const float* params, float* updates, void* mom_out, float* params_out,
                   void* stream);
int opt_sgd_bwd_ex(const opt_tree* tree, const opt_sgd_hp* hp, const opt_ext* ext,
                   int state_dtype, int compute, const float* g, const void* mom,
                   const float* params, const float* d_updates, const float* d_mom_out,
                   float* d_g, float* d_mom, float* d_params, double* d_hp, double* d_hp_leaf,
                   void* workspace, size_t workspace_bytes, void* stream);

/* ----------------------------------------- combining partial hyper sums
 * out[c] = sum over r = 0 .. rows-1 (in that order) of in[r * cols + c]:
 * the hyper-gradient sums of a step split into several calls (e.g. the
 * chunks of a host-streamed step, offload.py) combined on the device in a
 * fixed order (row a5; bitwise reproducible). in: device fp64 [rows][cols]
 * row-major (caller-owned); out: device fp64 [cols], written (not
 * accumulated); rows = 0 writes zeros. OPT_EINVAL on negative sizes or a
 * NULL pointer that is needed. */
int opt_sum_rows(int64_t rows, int64_t cols, const double* in, double* out, void* stream);

/* ----------------------------------- strided row copies (host streaming)
 * Plumbing of the host-streamed step (offload.py), ABI v6: copies `rows`
 * rows of `width_bytes` bytes, row r from src + r*spitch to dst + r*dpitch,
 * as ONE asynchronous DMA call on `stream` (cudaMemcpy2DAsync, direction
 * from the pointers: pinned host <-> device or device <-> device). Six
 * arrays' chunk moved this way takes one copy-engine command instead of six
 * (measured: both PCIe directions at once 6.3 ms vs 7.3 ms for 2 x 280 MB in
 * 8 chunks; profiles/r02bj_*). No arithmetic. Requires width_bytes <=
 * dpitch and <= spitch (when rows > 1); rows or width 0: nothing. Host
 * memory must be pinned for the copy to be asynchronous. OPT_EINVAL on a
 * bad size or NULL pointer, OPT_ECUDA if the copy cannot be enqueued. */
int opt_copy_rows(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width_bytes,
                  size_t rows, void* stream);

/* ------------------------------------------- apply_updates (row a8)
 * out = params + updates (out may alias params). Its VJP is the identity. */
int opt_apply_updates(int64_t numel, const float* params, const float* updates,
                      float* out, void* stream);

/* ------------------------------------- unrolled-sweep workload (row a9)
 * The synthetic inner loss of DESIGN.md "Input recipe" (C3), L_in =
 * 1/2 sum a_i (theta_i - phi_i)^2, whose gradient and Hessian-vector
 * product a real model would get from autograd:
 *   opt_quadratic_grad: g = a (theta - phi)
 *   opt_quadratic_rev:  theta_bar += a g_bar ;
 *                       phi_bar = (init_phi ? 0 : phi_bar) - a g_bar   (in place;
 *                       phi_bar is not read when init_phi != 0) */
int opt_quadratic_grad(int64_t numel, const float* a, const float* theta,
                       const float* phi, float* g, void* stream);
int opt_quadratic_rev(int64_t numel, const float* a, const float* g_bar,
                      float* theta_bar, float* phi_bar, int init_phi, void* stream);

/* Fused inner-loss glue (SV §8(f) NEXT-2: "fusing the inner-loss glue into
 * the step"): one unrolled step of the C3 sweep with the synthetic inner
 * loss L_in = 1/2 sum a (theta - phi)^2 folded into the Adam kernels.
 *   opt_adam_quad_fwd: g = a (theta - phi) -> g_out (NULL = not stored);
 *     Adam step on g (state as opt_adam_fwd); theta_out = theta + u.
 *     = opt_quadratic_grad + opt_adam_fwd(params=theta) in one pass.
 *   opt_adam_quad_rev: the Adam VJP at (g, mu, nu) with d_updates =
 *     theta_bar (cotangent of theta_out), then in place
 *     theta_bar += a d_g,  phi_bar = (init_phi ? 0 : phi_bar) - a d_g;
 *     d_mu/d_nu/d_hp as opt_adam_bwd; d_g itself is not stored.
 *     = opt_adam_bwd + opt_quadratic_rev in one pass.
 * theta_bar and phi_bar are read and written in place (exact aliasing). */
int opt_adam_quad_fwd(const opt_tree* tree, int64_t step, const opt_adam_hp* hp,
                      int state_dtype, int compute, const float* a, const float* phi,
                      const float* theta, const void* mu, const void* nu, float* g_out,
                      void* mu_out, void* nu_out, float* theta_out, void* stream);
int opt_adam_quad_rev(const opt_tree* tree, int64_t step, const opt_adam_hp* hp,
                      int state_dtype, int compute, const float* a, const float* g,
                      const void* mu, const void* nu, float* theta_bar, const float* d_mu_out,
                      const float* d_nu_out, float* d_mu, float* d_nu, float* phi_bar,
                      int init_phi, double* d_hp, void* workspace, size_t workspace_bytes,
                      void* stream);

/* ------------------------------------ zero-order ES (SV §8(f) NEXT-3)
 * PAPER.md §2.2 "Zero-order Differentiation (ZD)": ES optimises the
 * Gaussian smoothing f~(theta) = E_z[f(theta + sigma z)], z ~ N(0, I), with
 * gradient (1/sigma) E_z[f(theta + sigma z) z]. The noise z_ij is never
 * stored: it is a counter-based draw keyed on (seed, sample i, element j)
 * (reading N3 gives the exact definition), regenerated by both
 * calls.
 * opt_es_perturb writes the points the caller's black-box f is evaluated at:
 *   row r of `out` (row stride ld = numel rounded up to a multiple of 4
 *   floats) is theta + sigma z_(sample0 + i) for r = i (antithetic == 0), or
 *   theta + sigma z_i for r = 2i and theta - sigma z_i for r = 2i+1.
 *   out holds n_samples * (antithetic ? 2 : 1) * ld floats.
 * opt_es_grad: given f_values (device float, same row order, samples
 *   0..n_samples-1), grad = 1/(n sigma) sum_i f_i z_i (naive) or
 *   1/(2 n sigma) sum_i (f_(2i) - f_(2i+1)) z_i (antithetic).
 * n_samples <= 4096 per call; sigma > 0. theta/out/grad 16-byte aligned. */
int opt_es_perturb(int64_t numel, int64_t n_samples, int64_t sample0, int antithetic,
                   double sigma, uint64_t seed, const float* theta, float* out, void* stream);
int opt_es_grad(int64_t numel, int64_t n_samples, int antithetic, double sigma, uint64_t seed,
                const float* f_values, float* grad, void* stream);

/* ------------------------------ implicit-gradient solvers (SV §8(f) NEXT-4)
 * PAPER.md §2.2 "Implicit Gradient (IG)": the implicit function
 * theorem needs linear solves with dF/dtheta, by conjugate gradient (iMAML)
 * or a Neumann series. The matrix-vector product is the caller's (autograd
 * HVP/JVP); these calls are the rest of each iteration, fused, on flat fp32
 * vectors of n elements, with the scalars kept on the device in a
 * caller-owned double state[8] (state[0] = r.r, [1] = p.Ap, [2] = alpha,
 * [3] = beta, [4] = r0.r0, [5] = iterations) so no call synchronises:
 *   opt_cg_init:      r = b - Ax0 (Ax0 NULL: x0 = 0), p = r, rr = rr0 = r.r
 *   opt_cg_alpha:     pAp = p.Ap, alpha = rr / pAp (0 if pAp == 0)
 *   opt_cg_update:    x += alpha p, r -= alpha Ap, beta = r.r / rr, rr = r.r
 *   opt_cg_direction: p = r + beta p
 *   opt_neumann_step: v = v - alpha Av, x = x + v   (x = alpha sum (I - alpha A)^k b
 *                     when started from v = x = alpha b)
 * Dot products are fp64, deterministic (fixed grid and order). workspace:
 * >= opt_workspace_bytes of a one-leaf tree, zero-filled once. */
int opt_cg_init(int64_t n, const float* b, const float* Ax0, float* r, float* p, double* state,
                void* workspace, size_t workspace_bytes, void* stream);
int opt_cg_alpha(int64_t n, const float* p, const float* Ap, double* state, void* workspace,
                 size_t workspace_bytes, void* stream);
int opt_cg_update(int64_t n, float* x, float* r, const float* p, const float* Ap, double* state,
                  void* workspace, size_t workspace_bytes, void* stream);
int opt_cg_direction(int64_t n, float* p, const float* r, const double* state, void* stream);
int opt_neumann_step(int64_t n, float* v, const float* Av, float* x, double alpha, void* stream);

/* ------------------------------------- sharded step over peer memory
 * SURVEY §8(f) NEXT-2, element-sharded (ZeRO-1) Adam for W ranks of one
 * node, with the reduce-scatter, the fused step and the all-gather in ONE
 * kernel over peer memory (NVLink / NVSwitch loads and stores through
 * CUDA-IPC-mapped pointers) instead of two collectives around a local step.
 * Rank r owns elements [lo, lo + n_shard) of the flat tree. For each owned
 * element e:
 *   g      = grad_scale * sum_{w = 0..world-1} g_peers[w][e]   (fixed order)
 *   (u, m', v') = Adam_step(g, mu[e - lo], nu[e - lo])          (as opt_adam_fwd)
 *   theta' = params[e] + u, written to params_peers[w][e] for every w
 * mu / nu (fp32, the shard only) are updated in place. g_peers[w] /
 * params_peers[w] are device pointers valid in this process (the peer's
 * buffer mapped by CUDA IPC, or local memory); params is this rank's copy
 * (== params_peers[rank]). The caller orders the call: every peer's
 * gradient complete before, every peer's writes complete after (e.g. a
 * stream sync + process-group barrier on both sides). 1 <= world <=
 * OPT_MAX_PEERS; pointers 16-byte aligned; lo % 4 == 0. */
#define OPT_MAX_PEERS 8
typedef struct {
  const float* g[OPT_MAX_PEERS];
  float* params[OPT_MAX_PEERS];
} opt_peers;
int opt_adam_fwd_peers(int world, const opt_peers* peers, int64_t lo, int64_t n_shard,
                       int64_t step, const opt_adam_hp* hp, double grad_scale, float* mu,
                       float* nu, const float* params, void* stream);

/* Device-side barrier for opt_adam_fwd_peers (replaces a host stream sync
 * + process-group barrier on each side of the step). flags->f[w] is peer
 * w's flag array of 2 * OPT_MAX_PEERS uint64 (zero-initialised once, mapped
 * into this process by CUDA IPC for remote ranks; f[rank] is this rank's
 * own). One launch on `stream` (one warp): after a system-scope fence, it
 * writes `epoch` into slot `slot` (0 = gradients ready, 1 = parameter
 * stores done) of every peer's array at index slot * OPT_MAX_PEERS + rank,
 * then waits until every peer has written `epoch` (or more) into this
 * rank's array. Epochs increase by step (>= 1); the arrays are never
 * reset. The stream does not advance past the wait, so the order is:
 *   gradient -> signal_wait(0, t) -> opt_adam_fwd_peers -> signal_wait(1, t)
 * with no host round trip. A wait longer than timeout_s stops waiting and
 * sets *status (device int) to 1: the step's result is then undefined and
 * the caller should report it (no hang). */
typedef struct {
  uint64_t* f[OPT_MAX_PEERS];
} opt_peer_flags;
int opt_peer_signal_wait(int world, int rank, int slot, const opt_peer_flags* flags,
                         uint64_t epoch, double timeout_s, int* status, void* stream);

/* -------------------------------------------------------------- misc */
const char* opt_status_string(int status);
/* Message of the last failing call on this host thread ("" if none). */
const char* opt_last_error(void);
int opt_abi_version(void);
/* Kernel launches this library has enqueued in this process (all threads);
 * used by bench.py to report gpu_launches. */
int64_t opt_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* DIFFOPT_H */
