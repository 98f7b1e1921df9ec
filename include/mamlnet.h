/* include/mamlnet.h -- C ABI of the task-batched MAML network kernels (C4).
 *
 * What this is: the loss function a MAML meta-batch differentiates through
 * (reading Z16: 4 x [conv3x3(64) -> batch norm ->
 * ReLU -> 2x2 max-pool], fc -> 5 ways; MAML, "large
 * task-level batch size" P:25, distributed meta-batch P:269). It is the
 * WORKLOAD of the paper's optimizer hot path, not the method: the inner
 * SGD-momentum step and its VJP run in libdiffopt.so (include/diffopt.h).
 * The convolutions' forward and input-gradient contractions stay cuBLAS
 * batched SGEMMs; this library supplies the memory-bound layers around them
 * in one pass each, the hand-derived second derivative of the norm/pool
 * block that a second-order meta-gradient (create_graph, reading Z15) needs,
 * and a split-K fp32 kernel for the weight-gradient contraction (long n,
 * tiny output) that cuBLAS leaves under-parallel at a few tasks per GPU.
 *
 * Data layout: activations are task-major [T, C, B, H, W] fp32, contiguous.
 * A "group" g = t*C + c is one (task, channel) pair: its B*H*W elements are
 * contiguous at offset g*B*H*W, and batch-norm statistics are per group
 * (each task normalises over its own images). Per-group parameters (gamma,
 * beta) and per-group outputs are arrays of G = T*C floats indexed by g.
 * Pooled tensors are [T, C, B, H/2, W/2] (floor), codes one byte per pooled
 * element: 0..3 = window position (dy*2 + dx) of the maximum when the ReLU
 * is active (maximum > 0), 255 when it is not (zero output, zero gradient).
 *
 * Conventions: DEVICE pointers, fp32 unless stated; the caller owns every
 * buffer; no allocation, no synchronisation; all work enqueued on `stream`
 * (cudaStream_t, NULL = legacy default). Returns 0 (NET_OK), NET_EINVAL on a
 * bad size or NULL required pointer (nothing launched, message in
 * net_last_error()), NET_ECUDA on a launch error. Nullable inputs are
 * marked; NULL means zero. Group sums are fp64 in a fixed order (bitwise
 * reproducible run to run).
 */
#ifndef MAMLNET_H
#define MAMLNET_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MAMLNET_ABI_VERSION 3
#define NET_OK 0
#define NET_EINVAL 1
#define NET_ECUDA 3

/* 3x3, padding-1 im2col of h [G, B, H, W] (G = T*Cin) into
 * cols [G, 9, B, H, W], i.e. [T, Cin*9, B*H*W] with row cin*9 + 3i + j:
 * cols[g, 3i+j, b, y, x] = h[g, b, y+i-1, x+j-1] (0 outside the image). */
int net_im2col3x3(int64_t G, int64_t B, int64_t H, int64_t W, const float* h, float* cols,
                  void* stream);

/* Adjoint of net_im2col3x3: dh[g, b, y, x] = sum over (i, j) with the
 * source inside the image of cols[g, 3i+j, b, y-i+1, x-j+1]. Written, not
 * accumulated. */
int net_col2im3x3(int64_t G, int64_t B, int64_t H, int64_t W, const float* cols, float* dh,
                  void* stream);

/* Training-mode batch norm (biased batch variance, per group) + 2x2 max-pool
 * (floor) + ReLU, forward:
 *   mean_g = mean(x_g), rstd_g = 1/sqrt(var_g + eps),
 *   z = gamma_g * (x - mean_g) * rstd_g + beta_g,
 *   out[p] = max(0, max of z over window p), code[p] as above.
 * x [G,B,H,W] -> out [G,B,H/2,W/2], code (uint8, same shape), mean, rstd [G]
 * (saved for the backward). Requires H, W >= 2. */
int net_bnpool_fwd(int64_t G, int64_t B, int64_t H, int64_t W, const float* x,
                   const float* gamma, const float* beta, double eps, float* out, uint8_t* code,
                   float* mean, float* rstd, void* stream);

/* net_bnpool_fwd that also writes the next convolution's input columns:
 * cols [G, 9, B, H/2, W/2] = net_im2col3x3 of `out` (ABI v3; one launch
 * instead of two on the forward chain). Only positions whose source lies
 * inside the pooled map are written; the caller keeps the others (the
 * padding taps) zero, e.g. by zero-filling the buffer once. cols must not
 * be NULL. */
int net_bnpool_fwd_cols(int64_t G, int64_t B, int64_t H, int64_t W, const float* x,
                        const float* gamma, const float* beta, double eps, float* out,
                        uint8_t* code, float* mean, float* rstd, float* cols, void* stream);

/* VJP of net_bnpool_fwd. dy = the pooled cotangent dp routed to each window's
 * maximum (zero elsewhere and for inactive windows);
 *   dbeta_g = sum dy, dgamma_g = sum dy*xh  (xh = (x - mean) * rstd),
 *   dx = gamma*rstd*(dy - dbeta_g/n - xh*dgamma_g/n), n = B*H*W.
 * (The pool/ReLU mask is piecewise constant: no term of its own.) */
int net_bnpool_bwd(int64_t G, int64_t B, int64_t H, int64_t W, const float* dp,
                   const uint8_t* code, const float* x, const float* gamma, const float* mean,
                   const float* rstd, float* dx, float* dgamma, float* dbeta, void* stream);

/* VJP of net_bnpool_bwd (the second derivative a second-order meta-gradient
 * needs), given cotangents gdx [G,B,H,W], gdgamma [G], gdbeta [G] (each
 * nullable = 0) of its outputs, with dgamma/dbeta the values net_bnpool_bwd
 * returned. With A = dbeta/n, Bm = dgamma/n, r = rstd, G1 = sum gdx,
 * Gx = sum gdx*xh, GD = sum gdx*dy - A*G1 (per group):
 *   h      = -gamma*r*(dy*Gx/n + Bm*gdx) + gdgamma*dy
 *   g_x    = r*(h - mean(h) - xh*mean(h*xh)) - (gamma*r^2/n)*(GD - Bm*Gx)*xh
 *   g_dy   = gamma*r*(gdx - G1/n - xh*Gx/n) + gdgamma*xh + gdbeta
 *   g_dp   = g_dy at each active window's maximum (0 for inactive windows)
 *   g_gamma= r*(GD - Bm*Gx)
 * (derivation in DESIGN.md §8; checked against PyTorch's float64 double
 * backward of batch_norm/max_pool2d/relu in tests/test_mamlnet_gpu.py). */
int net_bnpool_bwd2(int64_t G, int64_t B, int64_t H, int64_t W, const float* gdx,
                    const float* gdgamma, const float* gdbeta, const float* dp,
                    const uint8_t* code, const float* x, const float* gamma, const float* mean,
                    const float* rstd, const float* dgamma, const float* dbeta, float* g_dp,
                    float* g_x, float* g_gamma, void* stream);

/* Batched "NT" product with a long contraction (the convolution
 * weight-gradient shape): C[t] = A[t] . B[t]^T, A [T, M, N], B [T, P, N],
 * C [T, M, P], all contiguous, fp32 arithmetic (fp32 FFMA accumulation over
 * each of S contiguous n-ranges, then the S partials summed in order;
 * S chosen from the sizes so that ~4 CTAs per SM exist). Workspace: a
 * device buffer of net_gemm_nt_workspace_bytes(T, M, P, N) bytes (0 means
 * none needed), caller-owned, contents irrelevant. N == 0 writes zeros.
 * Requires T <= 65535. */
size_t net_gemm_nt_workspace_bytes(int64_t T, int64_t M, int64_t P, int64_t N);
int net_gemm_nt(int64_t T, int64_t M, int64_t P, int64_t N, const float* A, const float* B,
                float* C, void* workspace, size_t workspace_bytes, void* stream);

/* As net_gemm_nt with a second operand pair and an accumulate flag:
 *   C[t] (+)= A[t].B[t]^T + A2[t].B2[t]^T
 * (A2, B2 both NULL = one pair; accumulate != 0 adds into C's contents).
 * Both pairs' n-ranges are one launch, then one fixed-order reduce over all
 * partials (bitwise reproducible). Workspace:
 * net_gemm_nt2_workspace_bytes(T, M, P, N, npairs, accumulate). Used for the
 * tangent of a convolution weight gradient, d(dy.cols^T) = dyd.cols^T +
 * dy.colsd^T, accumulated into a parameter cotangent. */
size_t net_gemm_nt2_workspace_bytes(int64_t T, int64_t M, int64_t P, int64_t N, int npairs,
                                    int accumulate);
int net_gemm_nt2(int64_t T, int64_t M, int64_t P, int64_t N, const float* A, const float* B,
                 const float* A2, const float* B2, float* C, int accumulate, void* workspace,
                 size_t workspace_bytes, void* stream);

/* ---- forward-mode derivatives (Hessian-vector products of the inner loss,
 * forward-over-reverse; the hand-scheduled MAML step) ---- */

/* JVP of net_bnpool_fwd at (x, gamma, beta) along (xd, gd, bd) (gd, bd
 * nullable = 0), with the forward's code/mean/rstd (routing is piecewise
 * constant: held fixed). Per group, with r = rstd, xh = (x - mean)*r:
 *   a = mean(xd), b = mean(xh*xd)                 -> s1[g] = a, s2[g] = b
 *   xhd = r*(xd - a - xh*b)                       (tangent of xh)
 *   outd[p] = gd*xh + gamma*xhd + bd at the window maximum of an active
 *             window p, 0 for inactive windows. */
int net_bnpool_jvp(int64_t G, int64_t B, int64_t H, int64_t W, const float* x, const float* xd,
                   const float* gamma, const float* gd, const float* bd, const uint8_t* code,
                   const float* mean, const float* rstd, float* outd, float* s1, float* s2,
                   void* stream);

/* net_bnpool_jvp that also writes cols = net_im2col3x3 of `outd` (the next
 * convolution's tangent columns), with net_bnpool_fwd_cols' convention:
 * padding taps are not written (kept zero by the caller). ABI v3. */
int net_bnpool_jvp_cols(int64_t G, int64_t B, int64_t H, int64_t W, const float* x,
                        const float* xd, const float* gamma, const float* gd, const float* bd,
                        const uint8_t* code, const float* mean, const float* rstd, float* outd,
                        float* s1, float* s2, float* cols, void* stream);

/* JVP of net_bnpool_bwd at (dp, x, gamma) along (dpd, xd, gd) (gd nullable),
 * given the backward's dgamma/dbeta and s1/s2 of net_bnpool_jvp for the same
 * xd. dy / dyd = dp / dpd routed to the window maxima. With A = dbeta/n,
 * Bm = dgamma/n, D = dy - A - xh*Bm (so dx = gamma*r*D) and xhd as above:
 *   dbetad  = sum dyd                   (ADDED to dbd_acc[g]; nullable)
 *   dgammad = sum (dyd*xh + dy*xhd)     (ADDED to dgd_acc[g]; nullable)
 *   Dd  = dyd - dbetad/n - xhd*Bm - xh*dgammad/n
 *   dxd = (gd*r - gamma*r^2*b)*D + gamma*r*Dd     (r' = -r^2*b) */
int net_bnpool_bwd_jvp(int64_t G, int64_t B, int64_t H, int64_t W, const float* dp,
                       const float* dpd, const uint8_t* code, const float* x, const float* xd,
                       const float* gamma, const float* gd, const float* mean, const float* rstd,
                       const float* dgamma, const float* dbeta, const float* s1, const float* s2,
                       float* dxd, float* dgd_acc, float* dbd_acc, void* stream);

/* Classifier head of T tasks, forward and backward in one launch (one CTA
 * per task): feat[t][b][c] = h4[t][c][b] (the [T, C, B] pooled map),
 * logits = feat.Wfc[t]^T + bfc[t] (Wfc [T, J, C], bfc [T, J]),
 * loss[t] = mean over b of cross_entropy(logits[b], labels[t][b]) (int64),
 * prob = softmax(logits) [T, B, J] (saved for the JVP), dl = (prob -
 * onehot)/B, dW[t] = dl^T.feat, db[t] = sum_b dl, dh4[t][c][b] =
 * (dl.Wfc)[b][c] (all written). */
int net_fc_xent(int64_t T, int64_t B, int64_t C, int64_t J, const float* h4, const float* Wfc,
                const float* bfc, const int64_t* labels, float* loss, float* prob, float* dW,
                float* db, float* dh4, void* stream);

/* JVP of net_fc_xent's (dW, db, dh4) along (h4d, Wd, bd) (each nullable = 0):
 *   ld = featd.Wfc^T + feat.Wd^T + bd;  dld = prob*(ld - sum_j prob*ld)/B
 *   dWd_acc[t] += dld^T.feat + dl^T.featd;  dbd_acc[t] += sum_b dld
 *   dh4d[t][c][b] = (dld.Wfc + dl.Wd)[b][c]  (written). */
int net_fc_xent_jvp(int64_t T, int64_t B, int64_t C, int64_t J, const float* h4, const float* h4d,
                    const float* Wfc, const float* Wd, const float* bd, const int64_t* labels,
                    const float* prob, float* dWd_acc, float* dbd_acc, float* dh4d,
                    void* stream);

/* Fold the task axis of a leaf-major T-task buffer: with per-task leaf
 * offsets off[0..n_leaves] (host and device copies, off[0] = 0, monotone),
 *   out[off[l] + i] = sum over t = 0..T-1 (in order) of in[T*off[l] + t*size_l + i].
 * (theta_0 of every task is phi, so phi's cotangent is this sum.) */
int net_task_sum(int64_t T, int64_t n_leaves, const int64_t* h_offsets, const int64_t* d_offsets,
                 const float* in, float* out, void* stream);

const char* net_last_error(void);
int net_abi_version(void);
int64_t net_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* MAMLNET_H */
