// abi.cu -- host side of the C ABI declared in include/diffopt.h.
//
// Validation, per-step scalar precompute in double,
// kernel selection (op x state dtype x compute precision x reduction mode)
// and launch on the caller's stream. No allocation, no synchronisation.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>
#include <unordered_map>

#include "diffopt.h"
#include "step_kernel.cuh"
#include "tma_kernel.cuh"

using namespace dopt;

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

constexpr int64_t kMaxGrid = 4096;       // upper bound on blocks of any launch
constexpr size_t kCounterBytes = 256;    // workspace head (ticket counter)
constexpr int kNhMax = 5;
constexpr int kDefaultCompute = OPT_COMPUTE_F32;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

bool misaligned(const void* p) { return p && (reinterpret_cast<uintptr_t>(p) & 15u); }

int check_align(std::initializer_list<const void*> ps) {
  int k = 0;
  for (const void* p : ps) {
    if (misaligned(p)) return fail(OPT_EALIGN, "array argument #%d (%p) is not 16-byte aligned", k, p);
    ++k;
  }
  return OPT_OK;
}

// Tree validation (row a1): offsets monotone, [0] = 0, [n] = numel.
int check_tree(const opt_tree* t) {
  if (!t) return fail(OPT_EINVAL, "tree is NULL");
  if (t->numel < 0) return fail(OPT_EINVAL, "numel < 0");
  if (t->n_leaves < 0) return fail(OPT_EINVAL, "n_leaves < 0");
  if (t->n_leaves > 0) {
    if (!t->h_offsets) return fail(OPT_EINVAL, "h_offsets is NULL with n_leaves > 0");
    if (t->h_offsets[0] != 0) return fail(OPT_EINVAL, "offsets[0] != 0");
    for (int64_t l = 0; l < t->n_leaves; ++l)
      if (t->h_offsets[l + 1] < t->h_offsets[l])
        return fail(OPT_EINVAL, "offsets decrease at leaf %lld", (long long)l);
    if (t->h_offsets[t->n_leaves] != t->numel)
      return fail(OPT_EINVAL, "offsets[n_leaves] = %lld != numel = %lld",
                  (long long)t->h_offsets[t->n_leaves], (long long)t->numel);
  }
  return OPT_OK;
}

// Leaf-mode workspace slots (doubles / kNhMax): piece partials (chunk +
// leaf slots), super-chunk partials, leaf_finalize block partials.
struct LeafSlots {
  int64_t part1, part2, blocks;
};
LeafSlots leaf_slots(const opt_tree* t) {
  const int64_t nl = t->n_leaves;
  return {n_chunks_of(t->numel) + nl, n_supers_of(t->numel) + nl, (nl + kWarps - 1) / kWarps};
}

bool finite(double x) { return std::isfinite(x); }
bool unit(double b) { return finite(b) && b >= 0.0 && b < 1.0; }

int resolve_compute(int compute, int* ct) {
  if (compute == OPT_COMPUTE_DEFAULT) compute = kDefaultCompute;
  if (compute != OPT_COMPUTE_F32 && compute != OPT_COMPUTE_F64)
    return fail(OPT_EINVAL, "compute = %d is not an opt_compute", compute);
  *ct = compute;
  return OPT_OK;
}

int check_state_dtype(int sd) {
  if (sd != OPT_F32 && sd != OPT_BF16)
    return fail(OPT_EINVAL, "state_dtype = %d is not an opt_state_dtype", sd);
  return OPT_OK;
}

// Per-device SM count and per-(kernel, smem) occupancy, queried once: the
// host path of a call is on the critical path of launch-bound workloads
// (small trees, MAML inner loops).
std::mutex g_cache_mu;
std::unordered_map<uint64_t, int> g_occ_cache;
std::atomic<int> g_sms[64];

int sm_count(int* sms) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail(OPT_ECUDA, "cudaGetDevice: %s", cudaGetErrorString(e));
  if (dev < 64) {
    int c = g_sms[dev].load(std::memory_order_relaxed);
    if (c > 0) {
      *sms = c;
      return OPT_OK;
    }
  }
  int c = 0;
  e = cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return fail(OPT_ECUDA, "device query failed: %s", cudaGetErrorString(e));
  if (dev < 64) g_sms[dev].store(c, std::memory_order_relaxed);
  *sms = c;
  return OPT_OK;
}

// Persistent grid: SMs x resident blocks of this kernel, capped by work.
template <class K>
int grid_for(K kernel, int64_t work_blocks, size_t smem, int* grid) {
  int sms = 0, per_sm = 0;
  int rc = sm_count(&sms);
  if (rc) return rc;
  const uint64_t key = reinterpret_cast<uint64_t>(reinterpret_cast<const void*>(kernel)) ^
                       ((uint64_t)smem << 48);
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_occ_cache.find(key);
    if (it != g_occ_cache.end()) per_sm = it->second;
  }
  if (per_sm == 0) {
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kBlock, smem);
    if (e != cudaSuccess) return fail(OPT_ECUDA, "occupancy query: %s", cudaGetErrorString(e));
    if (per_sm < 1) per_sm = 1;
    std::lock_guard<std::mutex> lk(g_cache_mu);
    g_occ_cache[key] = per_sm;
  }
  int64_t g = (int64_t)sms * per_sm;
  if (g > kMaxGrid) g = kMaxGrid;
  if (work_blocks < g) g = work_blocks;
  *grid = (int)(g > 0 ? g : 1);
  return OPT_OK;
}

#ifndef DOPT_PDL
#define DOPT_PDL 1
#endif
// Launch with programmatic dependent launch (PDL): the grid may be scheduled
// while the previous kernel on the stream drains; every step kernel starts
// with griddepcontrol.wait, so it still observes all prior work.
template <class K, class... Args>
cudaError_t launch_k(K kernel, int grid, int block, size_t smem, cudaStream_t s, Args... args) {
#if DOPT_PDL
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
#else
  kernel<<<grid, block, smem, s>>>(args...);
  return cudaGetLastError();
#endif
}

#define TRY(x)                \
  do {                        \
    int rc_ = (x);            \
    if (rc_) return rc_;      \
  } while (0)

int launched(cudaStream_t) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(OPT_ECUDA, "kernel launch failed: %s", cudaGetErrorString(e));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return OPT_OK;
}

// Workspace and reduction plumbing shared by the three backward ops.
// Reduction / leaf-mode plumbing of one launch. Leaf mode (chunks split at
// leaf boundaries, step_kernel.cuh) is used when per-leaf outputs or
// per-leaf learning rates are requested.
struct Reduce {
  double* d_hp;
  double* d_hp_leaf;
  const float* lr_leaf;
  bool leaf;
  double* partials;      // uniform: per block; leaf: per piece slot
  unsigned int* counter;
  double* part2;         // leaf mode: super-chunk slots
  double* block_part;    // leaf mode: leaf_finalize block partials
};

int setup_reduce(const opt_tree* t, double* d_hp, double* d_hp_leaf, const float* lr_leaf,
                 void* ws, size_t ws_bytes, Reduce* r) {
  r->d_hp = d_hp;
  r->d_hp_leaf = d_hp_leaf;
  r->lr_leaf = lr_leaf;
  r->leaf = d_hp_leaf != nullptr || lr_leaf != nullptr;
  r->partials = nullptr;
  r->counter = nullptr;
  r->part2 = nullptr;
  r->block_part = nullptr;
  if (r->leaf) {
    if (t->n_leaves < 1) return fail(OPT_EINVAL, "per-leaf outputs/lr need n_leaves >= 1");
    if (!t->d_offsets) return fail(OPT_EINVAL, "per-leaf outputs/lr need tree->d_offsets");
  }
  if (!d_hp && !d_hp_leaf) return OPT_OK;
  size_t need = opt_workspace_bytes(t, r->leaf ? 1 : 0);
  if (!ws || ws_bytes < need)
    return fail(OPT_EWORKSPACE, "workspace %p of %zu bytes; need %zu", ws, ws_bytes, need);
  if (reinterpret_cast<uintptr_t>(ws) & 15u) return fail(OPT_EALIGN, "workspace not 16-byte aligned");
  r->counter = static_cast<unsigned int*>(ws);
  r->partials = reinterpret_cast<double*>(static_cast<char*>(ws) + kCounterBytes);
  if (r->leaf) {
    const LeafSlots ls = leaf_slots(t);
    r->part2 = r->partials + kNhMax * ls.part1;
    r->block_part = r->part2 + kNhMax * ls.part2;
  }
  return OPT_OK;
}

int zero_outputs(const opt_tree* t, int nh, double* d_hp, double* d_hp_leaf, cudaStream_t s) {
  cudaError_t e = cudaSuccess;
  if (d_hp) e = cudaMemsetAsync(d_hp, 0, sizeof(double) * nh, s);
  if (e == cudaSuccess && d_hp_leaf && t->n_leaves > 0)
    e = cudaMemsetAsync(d_hp_leaf, 0, sizeof(double) * nh * t->n_leaves, s);
  if (e != cudaSuccess) return fail(OPT_ECUDA, "cudaMemsetAsync: %s", cudaGetErrorString(e));
  return OPT_OK;
}

// Launch shape per direction: U vectors in flight per thread, MINB resident
// blocks per SM requested from ptxas (register cap). Tuned on B200
// (DESIGN.md "Kernels"); -D overrides exist for tuning sweeps.
#ifndef DOPT_U_FWD
#define DOPT_U_FWD 1
#endif
#ifndef DOPT_MINB_FWD
#define DOPT_MINB_FWD 1
#endif
#ifndef DOPT_U_BWD
#define DOPT_U_BWD 1
#endif
#ifndef DOPT_MINB_BWD
#define DOPT_MINB_BWD 3
#endif
#ifndef DOPT_U_FWD_BF16
#define DOPT_U_FWD_BF16 DOPT_U_FWD
#endif
#ifndef DOPT_U_BWD_BF16
#define DOPT_U_BWD_BF16 DOPT_U_BWD
#endif

// cp.async double-buffered streaming kernel (step_pipe)
#ifndef DOPT_FWD_GRID_MULT  // forward grid = persistent grid x this (0 = one block per 256 vectors)
#define DOPT_FWD_GRID_MULT 0
#endif
#ifndef DOPT_BWD_GRID_MULT  // backward grid = persistent grid x this (0 = kMaxGrid), <= kMaxGrid
#define DOPT_BWD_GRID_MULT 1
#endif
#ifndef DOPT_PIPE_FWD
#define DOPT_PIPE_FWD 0
#endif
#ifndef DOPT_PIPE_BWD
#define DOPT_PIPE_BWD 0
#endif
#ifndef DOPT_TMA_FWD
#define DOPT_TMA_FWD 0
#endif
#ifndef DOPT_TMA_BWD
#define DOPT_TMA_BWD 0
#endif

// TMA-bulk pipelined path: one CTA per SM, STAGES-deep smem ring.
#ifndef DOPT_TMA_NCONS
#define DOPT_TMA_NCONS 256
#endif
#ifndef DOPT_TMA_CTAS
#define DOPT_TMA_CTAS 1
#endif
template <class Op, class ST>
int launch_tma(const Op& op, StepArgs<Op::NIN, Op::NOUT>& a, cudaStream_t s) {
  constexpr int NCONS = DOPT_TMA_NCONS, CTAS = DOPT_TMA_CTAS;
  constexpr uint32_t sb = TmaLayout<Op, ST, NCONS>::stage_bytes();
  constexpr uint32_t budget = 200 * 1024 / CTAS;
  constexpr int STAGES = (budget / sb) > 8 ? 8 : (int)(budget / sb);
  static_assert(STAGES >= 2, "TMA ring needs >= 2 stages");
  constexpr int kTmaTile = 4 * NCONS;
  auto k = step_tma<Op, ST, STAGES, NCONS, CTAS>;
  const size_t smem = tma_smem_bytes<Op, ST, STAGES, NCONS>();
  static const cudaError_t attr =  // once per instantiation (thread-safe static init)
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (attr != cudaSuccess) return fail(OPT_ECUDA, "smem attribute: %s", cudaGetErrorString(attr));
  int sms = 0;
  int rc = sm_count(&sms);
  if (rc) return rc;
  const int64_t tiles = (a.numel + kTmaTile - 1) / kTmaTile;
  int grid = (int)(tiles < (int64_t)sms * CTAS ? tiles : (int64_t)sms * CTAS);
  cudaError_t le = launch_k(k, grid > 0 ? grid : 1, NCONS + 32, smem, s, op, a);
  if (le != cudaSuccess) return fail(OPT_ECUDA, "launch: %s", cudaGetErrorString(le));
  return launched(s);
}

// fp64 arithmetic needs more registers: cap at 2 blocks/SM (128 regs) there
// instead of spilling under the fp32 cap.
template <class Op>
constexpr int minb_bwd() {
  return sizeof(typename Op::CT) == 8 ? (DOPT_MINB_BWD < 2 ? DOPT_MINB_BWD : 2) : DOPT_MINB_BWD;
}

template <class Op, bool kBwd>
constexpr int minb_for() {
  return kBwd ? minb_bwd<Op>() : DOPT_MINB_FWD;
}

// Launch one op: leaf mode, TMA variant or the uniform streaming kernel.
template <class Op, class ST, int U, int MINB, bool kTma, bool kPipe>
int launch(const Op& op, StepArgs<Op::NIN, Op::NOUT>& a, const Reduce& r, const opt_tree* t,
           cudaStream_t s) {
  a.d_hp = r.d_hp;
  a.d_hp_leaf = r.d_hp_leaf;
  a.partials = r.partials;
  a.counter = r.counter;
  a.lr_leaf = r.lr_leaf;
  a.want_hp = (r.d_hp || r.d_hp_leaf) ? 1 : 0;
  if (r.leaf) {
    a.offsets = t->d_offsets;
    a.n_leaves = t->n_leaves;
    auto k = step_leaf<Op, ST, U, MINB>;
    const size_t smem =
        t->n_leaves <= kMaxLeafSmem ? sizeof(int64_t) * (size_t)(t->n_leaves + 1) : 0;
    static const cudaError_t attr = cudaFuncSetAttribute(
        k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(int64_t) * (kMaxLeafSmem + 1)));
    if (attr != cudaSuccess) return fail(OPT_ECUDA, "smem attribute: %s", cudaGetErrorString(attr));
    int grid = 0;
    int rc = grid_for(k, (n_chunks_of(a.numel) + kWarps - 1) / kWarps, smem, &grid);
    if (rc) return rc;
    cudaError_t le = launch_k(k, grid, kBlock, smem, s, op, a);
    if (le != cudaSuccess) return fail(OPT_ECUDA, "launch: %s", cudaGetErrorString(le));
    TRY(launched(s));
    if constexpr (Op::NH > 0) {
      if (a.want_hp) {  // piece slots -> super-chunk slots -> per-leaf and global sums
        constexpr int NH = Op::NH;
        const int64_t fold_blocks = (n_supers_of(a.numel) + kWarps - 1) / kWarps;
        le = launch_k(leaf_fold<NH>, (int)fold_blocks, kBlock, 0, s, (const double*)r.partials,
                      t->d_offsets, t->n_leaves, a.numel, r.part2);
        if (le != cudaSuccess) return fail(OPT_ECUDA, "launch: %s", cudaGetErrorString(le));
        TRY(launched(s));
        const int fg = (int)((t->n_leaves + kWarps - 1) / kWarps);
        le = launch_k(leaf_finalize<NH>, fg, kBlock, 0, s, (const double*)r.part2, t->d_offsets,
                      t->n_leaves, r.d_hp_leaf, r.d_hp, r.block_part, r.counter);
        if (le != cudaSuccess) return fail(OPT_ECUDA, "launch: %s", cudaGetErrorString(le));
        TRY(launched(s));
      }
    }
    return OPT_OK;
  }
  if (kTma) return launch_tma<Op, ST>(op, a, s);
  if constexpr (kPipe) {
    auto k = step_pipe<Op, ST, MINB>;
    const size_t smem = sizeof(float4) * 2 * Op::NIN * kBlock;
    static const cudaError_t attr =
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (attr != cudaSuccess) return fail(OPT_ECUDA, "smem attribute: %s", cudaGetErrorString(attr));
    int grid = 0;
    int64_t work = ((a.numel >> 2) + kBlock - 1) / kBlock + 1;
    int rc = grid_for(k, work, smem, &grid);
    if (rc) return rc;
    cudaError_t le = launch_k(k, grid, kBlock, smem, s, op, a);
    if (le != cudaSuccess) return fail(OPT_ECUDA, "launch: %s", cudaGetErrorString(le));
    return launched(s);
  }
  auto k = step_uniform<Op, ST, U, MINB>;
  int grid = 0;
  int64_t work = ((a.numel >> 2) + kBlock - 1) / kBlock + 1;
  int rc = grid_for(k, work, 0, &grid);
  if (rc) return rc;
  if constexpr (Op::NH == 0 && std::is_same<ST, float>::value) {
    // fp32 state and no block partials, so the grid is free: one block per
    // 256 vectors (measured on B200: fp32 forwards 103-106% of the copy peak
    // at 2^26-2^30 vs 91-94% with the persistent grid, whose per-block tails
    // end unevenly; bf16-state forwards measured 2-5% slower this way, so they
    // keep the persistent grid; DOPT_FWD_GRID_MULT)
    int64_t g = DOPT_FWD_GRID_MULT > 0 ? (int64_t)grid * DOPT_FWD_GRID_MULT : work;
    if (g > work) g = work;
    if (g > 0x7FFFFFFF) g = 0x7FFFFFFF;
    grid = (int)g;
  } else if constexpr (Op::NH > 0) {
    int64_t g = DOPT_BWD_GRID_MULT > 0 ? (int64_t)grid * DOPT_BWD_GRID_MULT : kMaxGrid;
    if (g > kMaxGrid) g = kMaxGrid;  // block partials live in the workspace
    if (g > work) g = work;
    grid = (int)g;
  }
  cudaError_t le = launch_k(k, grid, kBlock, 0, s, op, a);
  if (le != cudaSuccess) return fail(OPT_ECUDA, "launch: %s", cudaGetErrorString(le));
  return launched(s);
}

// Dispatch on (state dtype, compute precision).
template <template <class> class OpT, bool kBwd, class Fill>
int dispatch(int state_dtype, int ct, StepArgs<OpT<float>::NIN, OpT<float>::NOUT>& a,
             const Reduce& r, const opt_tree* t, cudaStream_t s, Fill fill) {
  constexpr int U = kBwd ? DOPT_U_BWD : DOPT_U_FWD;
  // bf16 state moves 8-byte vectors: more of them in flight per thread
  constexpr int UB = kBwd ? DOPT_U_BWD_BF16 : DOPT_U_FWD_BF16;
  constexpr bool TMA = kBwd ? (DOPT_TMA_BWD != 0) : (DOPT_TMA_FWD != 0);
  constexpr bool PIPE = kBwd ? (DOPT_PIPE_BWD != 0) : (DOPT_PIPE_FWD != 0);
  if (ct == OPT_COMPUTE_F64) {
    OpT<double> op;
    fill(op);
    constexpr int MB = minb_for<OpT<double>, kBwd>();
    if (state_dtype == OPT_BF16)
      return launch<OpT<double>, bf16, U, MB, TMA, PIPE>(op, a, r, t, s);
    return launch<OpT<double>, float, U, MB, TMA, PIPE>(op, a, r, t, s);
  }
  OpT<float> op;
  fill(op);
  constexpr int MB = minb_for<OpT<float>, kBwd>();
  if (state_dtype == OPT_BF16) return launch<OpT<float>, bf16, UB, MB, TMA, PIPE>(op, a, r, t, s);
  return launch<OpT<float>, float, U, MB, TMA, PIPE>(op, a, r, t, s);
}

// b^t by repeated squaring in double (exact integer power).
double ipow(double b, int64_t t) {
  double r = 1.0, x = b;
  while (t > 0) {
    if (t & 1) r *= x;
    x *= x;
    t >>= 1;
  }
  return r;
}

int check_adam(int64_t step, const opt_adam_hp* hp) {
  if (!hp) return fail(OPT_EINVAL, "hp is NULL");
  if (step < 1) return fail(OPT_EINVAL, "step = %lld < 1", (long long)step);
  if (!finite(hp->lr)) return fail(OPT_EINVAL, "lr is not finite");
  if (!unit(hp->b1)) return fail(OPT_EINVAL, "b1 = %g outside [0, 1)", hp->b1);
  if (!unit(hp->b2)) return fail(OPT_EINVAL, "b2 = %g outside [0, 1)", hp->b2);
  if (!(finite(hp->eps) && hp->eps >= 0)) return fail(OPT_EINVAL, "eps = %g < 0", hp->eps);
  if (!(finite(hp->eps_root) && hp->eps_root >= 0))
    return fail(OPT_EINVAL, "eps_root = %g < 0", hp->eps_root);
  return OPT_OK;
}

int check_rms(const opt_rmsprop_hp* hp) {
  if (!hp) return fail(OPT_EINVAL, "hp is NULL");
  if (!finite(hp->lr)) return fail(OPT_EINVAL, "lr is not finite");
  if (!unit(hp->alpha)) return fail(OPT_EINVAL, "alpha = %g outside [0, 1)", hp->alpha);
  if (!(finite(hp->eps) && hp->eps >= 0)) return fail(OPT_EINVAL, "eps = %g < 0", hp->eps);
  return OPT_OK;
}

int check_sgd(const opt_sgd_hp* hp) {
  if (!hp) return fail(OPT_EINVAL, "hp is NULL");
  if (!finite(hp->lr)) return fail(OPT_EINVAL, "lr is not finite");
  if (!unit(hp->momentum)) return fail(OPT_EINVAL, "momentum = %g outside [0, 1)", hp->momentum);
  return OPT_OK;
}



// Per-step constants of each op (row a2): computed in double, rounded once
// to the compute type CT (reading Z8).
template <class Op>
void fill_adam_fwd(Op& op, int64_t step, const opt_adam_hp* hp) {
  typedef typename Op::CT CT;
  const double b1 = hp->b1, b2 = hp->b2;
  const double bc1 = 1.0 - ipow(b1, step), bc2 = 1.0 - ipow(b2, step);
  op.b1 = (CT)b1; op.om1 = (CT)(1.0 - b1); op.b2 = (CT)b2; op.om2 = (CT)(1.0 - b2);
  op.ibc1 = (CT)(1.0 / bc1); op.ibc2 = (CT)(1.0 / bc2); op.lr = (CT)hp->lr;
  op.eps = (CT)hp->eps; op.eps_root = (CT)hp->eps_root;
}

template <class Op>
void fill_adam_bwd(Op& op, int64_t step, const opt_adam_hp* hp) {
  typedef typename Op::CT CT;
  const double b1 = hp->b1, b2 = hp->b2, t = (double)step;
  const double p1 = ipow(b1, step), p2 = ipow(b2, step);
  const double p1m = ipow(b1, step - 1), p2m = ipow(b2, step - 1);
  const double bc1 = 1.0 - p1, bc2 = 1.0 - p2;
  // d mhat/d b1 = m K1 - g K2 ; d vhat/d b2 = v K3 - g^2 K4
  const double K1 = (1.0 - p1 + t * p1) / (bc1 * bc1);
  const double K2 = (1.0 - p1 - t * p1m * (1.0 - b1)) / (bc1 * bc1);
  const double K3 = (1.0 - p2 + t * p2) / (bc2 * bc2);
  const double K4 = (1.0 - p2 - t * p2m * (1.0 - b2)) / (bc2 * bc2);
  op.b1 = (CT)b1; op.om1 = (CT)(1.0 - b1); op.b2 = (CT)b2; op.two_om2 = (CT)(2.0 * (1.0 - b2));
  op.A = (CT)((1.0 - b1) / bc1); op.C = (CT)((1.0 - b2) / bc2);
  op.b1ibc1 = (CT)(b1 / bc1); op.b2ibc2 = (CT)(b2 / bc2);
  op.eps_root = (CT)hp->eps_root; op.lr = (CT)hp->lr; op.eps = (CT)hp->eps;
  op.Aeps = (CT)((1.0 - b1) / bc1 * hp->eps);
  op.kM = (CT)(b1 * hp->lr / bc1); op.kV = (CT)(0.5 * b2 * hp->lr / bc2);
  op.hlr = (CT)(0.5 * hp->lr);
  op.kM0 = (CT)(b1 / bc1); op.kV0 = (CT)(0.5 * b2 / bc2);
  op.K1 = (CT)K1; op.K2 = (CT)K2; op.K3 = (CT)K3; op.K4 = (CT)K4;
}

template <class Op>
void fill_rms_fwd(Op& op, const opt_rmsprop_hp* hp) {
  typedef typename Op::CT CT;
  op.alpha = (CT)hp->alpha; op.oma = (CT)(1.0 - hp->alpha); op.lr = (CT)hp->lr;
  op.eps = (CT)hp->eps;
}

template <class Op>
void fill_rms_bwd(Op& op, const opt_rmsprop_hp* hp) {
  typedef typename Op::CT CT;
  op.alpha = (CT)hp->alpha; op.oma = (CT)(1.0 - hp->alpha);
  op.two_oma = (CT)(2.0 * (1.0 - hp->alpha)); op.lr = (CT)hp->lr; op.eps = (CT)hp->eps;
  op.hlr = (CT)(0.5 * hp->lr);
}

template <class Op>
void fill_sgd(Op& op, const opt_sgd_hp* hp) {
  typedef typename Op::CT CT;
  op.lr = (CT)hp->lr; op.mu = (CT)hp->momentum; op.nesterov = hp->nesterov ? 1 : 0;
}

template <class Op>
void fill_ext(Op& op, const opt_ext* e, bool adam) {
  typedef typename Op::CT CT;
  op.wd = (CT)e->weight_decay;
  op.decoupled = (adam && e->decoupled) ? 1 : 0;
  op.maximize = e->maximize ? 1 : 0;
}

int check_rms_cm(const opt_rmsprop_cm_hp* hp) {
  if (!hp) return fail(OPT_EINVAL, "hp is NULL");
  if (!finite(hp->lr)) return fail(OPT_EINVAL, "lr is not finite");
  if (!unit(hp->alpha)) return fail(OPT_EINVAL, "alpha = %g outside [0, 1)", hp->alpha);
  if (!(finite(hp->eps) && hp->eps >= 0)) return fail(OPT_EINVAL, "eps = %g < 0", hp->eps);
  if (!unit(hp->momentum)) return fail(OPT_EINVAL, "momentum = %g outside [0, 1)", hp->momentum);
  return OPT_OK;
}

template <class Op>
void fill_rms_cm(Op& op, const opt_rmsprop_cm_hp* hp, const opt_ext* e) {
  typedef typename Op::CT CT;
  op.alpha = (CT)hp->alpha; op.oma = (CT)(1.0 - hp->alpha); op.lr = (CT)hp->lr;
  op.eps = (CT)hp->eps; op.mu = (CT)hp->momentum; op.centered = hp->centered ? 1 : 0;
  op.wd = (CT)e->weight_decay; op.maximize = e->maximize ? 1 : 0;
}

int check_ext(const opt_ext* e, const float* params, const opt_tree* t) {
  if (!e) return fail(OPT_EINVAL, "ext is NULL");
  if (!(finite(e->weight_decay) && e->weight_decay >= 0))
    return fail(OPT_EINVAL, "weight_decay = %g < 0", e->weight_decay);
  if (e->weight_decay != 0.0 && !params && t->numel > 0)
    return fail(OPT_EINVAL, "weight_decay != 0 needs params");
  if (misaligned(e->lr_leaf)) return fail(OPT_EALIGN, "lr_leaf not 16-byte aligned");
  return OPT_OK;
}

}  // namespace

extern "C" {

size_t opt_workspace_bytes(const opt_tree* tree, int per_leaf) {
  if (check_tree(tree)) return 0;
  int64_t slots = kMaxGrid;
  if (per_leaf) {
    const LeafSlots ls = leaf_slots(tree);
    const int64_t leaf = ls.part1 + ls.part2 + ls.blocks;
    if (leaf > slots) slots = leaf;
  }
  return kCounterBytes + sizeof(double) * kNhMax * (size_t)slots;
}

// ------------------------------------------------------------------ Adam
int opt_adam_fwd(const opt_tree* tree, int64_t step, const opt_adam_hp* hp, int state_dtype,
                 int compute, const float* g, const void* mu, const void* nu, float* updates,
                 void* mu_out, void* nu_out, const float* params, float* params_out,
                 void* stream) {
  g_err.clear();
  int ct = 0;
  TRY(check_tree(tree));
  TRY(check_adam(step, hp));
  TRY(check_state_dtype(state_dtype));
  TRY(resolve_compute(compute, &ct));
  TRY(check_align({g, mu, nu, updates, mu_out, nu_out, params, params_out}));
  if (tree->numel == 0) return OPT_OK;
  if (!g) return fail(OPT_EINVAL, "g is NULL");
  StepArgs<4, 4> a{};
  a.in[0] = g; a.in[1] = mu; a.in[2] = nu; a.in[3] = (params && params_out) ? params : nullptr;
  a.out[0] = updates; a.out[1] = mu_out; a.out[2] = nu_out;
  a.out[3] = (params && params_out) ? params_out : nullptr;
  a.numel = tree->numel;
  return dispatch<AdamFwd, false>(state_dtype, ct, a, Reduce{}, tree,
                                  static_cast<cudaStream_t>(stream),
                                  [&](auto& op) { fill_adam_fwd(op, step, hp); });
}

int opt_adam_bwd(const opt_tree* tree, int64_t step, const opt_adam_hp* hp, int state_dtype,
                 int compute, const float* g, const void* mu, const void* nu,
                 const float* d_updates, const float* d_mu_out, const float* d_nu_out,
                 float* d_g, float* d_mu, float* d_nu, double* d_hp, double* d_hp_leaf,
                 void* workspace, size_t workspace_bytes, void* stream) {
  g_err.clear();
  int ct = 0;
  TRY(check_tree(tree));
  TRY(check_adam(step, hp));
  TRY(check_state_dtype(state_dtype));
  TRY(resolve_compute(compute, &ct));
  TRY(check_align({g, mu, nu, d_updates, d_mu_out, d_nu_out, d_g, d_mu, d_nu}));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (tree->numel == 0) return zero_outputs(tree, 4, d_hp, d_hp_leaf, s);
  if (!g) return fail(OPT_EINVAL, "g is NULL");
  Reduce r;
  TRY(setup_reduce(tree, d_hp, d_hp_leaf, nullptr, workspace, workspace_bytes, &r));
  StepArgs<6, 3> a{};
  a.in[0] = g; a.in[1] = mu; a.in[2] = nu; a.in[3] = d_updates; a.in[4] = d_mu_out;
  a.in[5] = d_nu_out;
  a.out[0] = d_g; a.out[1] = d_mu; a.out[2] = d_nu;
  a.numel = tree->numel;
  return dispatch<AdamBwd, true>(state_dtype, ct, a, r, tree, s,
                                 [&](auto& op) { fill_adam_bwd(op, step, hp); });
}

int opt_adam_fwd_ex(const opt_tree* tree, int64_t step, const opt_adam_hp* hp,
                    const opt_ext* ext, int state_dtype, int compute, const float* g,
                    const void* mu, const void* nu, const float* params, float* updates,
                    void* mu_out, void* nu_out, float* params_out, void* stream) {
  g_err.clear();
  int ct = 0;
  TRY(check_tree(tree));
  TRY(check_adam(step, hp));
  TRY(check_ext(ext, params, tree));
  TRY(check_state_dtype(state_dtype));
  TRY(resolve_compute(compute, &ct));
  TRY(check_align({g, mu, nu, params, updates, mu_out, nu_out, params_out}));
  if (tree->numel == 0) return OPT_OK;
  if (!g) return fail(OPT_EINVAL, "g is NULL");
  Reduce r;
  TRY(setup_reduce(tree, nullptr, nullptr, ext->lr_leaf, nullptr, 0, &r));
  StepArgs<4, 4> a{};
  a.in[0] = g; a.in[1] = mu; a.in[2] = nu; a.in[3] = params;
  a.out[0] = updates; a.out[1] = mu_out; a.out[2] = nu_out;
  a.out[3] = params ? params_out : nullptr;
  a.numel = tree->numel;
  return dispatch<AdamFwdEx, false>(state_dtype, ct, a, r, tree, static_cast<cudaStream_t>(stream),
                                    [&](auto& op) {
                                      fill_adam_fwd(op.base, step, hp);
                                      fill_ext(op, ext, true);
                                    });
}

int opt_adam_bwd_ex(const opt_tree* tree, int64_t step, const opt_adam_hp* hp,
                    const opt_ext* ext, int state_dtype, int compute, const float* g,
                    const void* mu, const void* nu, const float* params, const float* d_updates,
                    const float* d_mu_out, const float* d_nu_out, float* d_g, float* d_mu,
                    float* d_nu, float* d_params, double* d_hp, double* d_hp_leaf,
                    void* workspace, size_t workspace_bytes, void* stream) {
  g_err.clear();
  int ct = 0;
  TRY(check_tree(tree));
  TRY(check_adam(step, hp));
  TRY(check_ext(ext, params, tree));
  TRY(check_state_dtype(state_dtype));
  TRY(resolve_compute(compute, &ct));
  TRY(check_align({g, mu, nu, params, d_updates, d_mu_out, d_nu_out, d_g, d_mu, d_nu, d_params}));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (tree->numel == 0) return zero_outputs(tree, 5, d_hp, d_hp_leaf, s);
  if (!g) return fail(OPT_EINVAL, "g is NULL");
  Reduce r;
  TRY(setup_reduce(tree, d_hp, d_hp_leaf, ext->lr_leaf, workspace, workspace_bytes, &r));
  StepArgs<7, 4> a{};
  a.in[0] = g; a.in[1] = mu; a.in[2] = nu; a.in[3] = params; a.in[4] = d_updates;
  a.in[5] = d_mu_out; a.in[6] = d_nu_out;
  a.out[0] = d_g; a.out[1] = d_mu; a.out[2] = d_nu; a.out[3] = d_params;
  a.numel = tree->numel;
  return dispatch<AdamBwdEx, true>(state_dtype, ct, a, r, tree, s, [&](auto& op) {
    fill_adam_bwd(op.base, step, hp);
    fill_ext(op, ext, true);
  });
}

// --------------------------------------------------------------- RMSProp
int opt_rmsprop_fwd(const opt_tree* tree, const opt_rmsprop_hp* hp, int state_dtype,
                    int compute, const float* g, const void* nu, float* updates, void* nu_out,
                    const float* params, float* params_out, void* stream) {
  g_err.clear();
  int ct = 0;
  TRY(check_tree(tree));
  TRY(check_rms(hp));
  TRY(check_state_dtype(state_dtype));
  TRY(resolve_compute(compute, &ct));
  TRY(check_align({g, nu, updates, nu_out, params, params_out}));
  if (tree->numel == 0) return OPT_OK;
  if (!g) return fail(OPT_EINVAL, "g is NULL");
  StepArgs<3, 3> a{};
  a.in[0] = g; a.in[1] = nu; a.in[2] = (params && params_out) ? params : nullptr;
  a.out[0] = updates; a.out[1] = nu_out; a.out[2] = (params && params_out) ? params_out : nullptr;
  a.numel = tree->numel;
  return dispatch<RmsFwd, false>(state_dtype, ct, a, Reduce{}, tree,
                                 static_cast<cudaStream_t>(stream),
                                 [&](auto& op) { fill_rms_fwd(op, hp); });
}

int opt_rmsprop_bwd(const opt_tree* tree, const opt_rmsprop_hp* hp, int state_dtype,
                    int compute, const float* g, const void* nu, const float* d_updates,
                    const float* d_nu_out, float* d_g, float* d_nu, double* d_hp,
                    double* d_hp_leaf, void* workspace, size_t workspace_bytes, void* stream) {
  g_err.clear();
  int ct = 0;
  TRY(check_tree(tree));
  TRY(check_rms(hp));
  TRY(check_state_dtype(state_dtype));
  TRY(resolve_compute(compute, &ct));
  TRY(check_align({g, nu, d_updates, d_nu_out, d_g, d_nu}));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (tree->numel == 0) return zero_outputs(tree, 3, d_hp, d_hp_leaf, s);
  if (!g) return fail(OPT_EINVAL, "g is NULL");
  Reduce r;
  TRY(setup_reduce(tree, d_hp, d_hp_leaf, nullptr, workspace, workspace_bytes, &r));
  StepArgs<4, 2> a{};
  a.in[0] = g; a.in[1] = nu; a.in[2] = d_updates; a.in[3] = d_nu_out;
  a.out[0] = d_g; a.out[1] = d_nu;
  a.numel = tree->numel;
  return dispatch<RmsBwd, true>(state_dtype, ct, a, r, tree, s,
                                [&](auto& op) { fill_rms_bwd(op, hp); });
}

int opt_rmsprop_fwd_ex(const opt_tree* tree, const opt_rmsprop_hp* hp, const opt_ext* ext,
                       int state_dtype, int compute, const float* g, const void* nu,
                       const float* params, float* updates, void* nu_out, float* params_out,
                       void* stream) {
  g_err.clear();
  int ct = 0;
  TRY(check_tree(tree));
  TRY(check_rms(hp));
  TRY(check_ext(ext, params, tree));
  TRY(check_state_dtype(state_dtype));
  TRY(resolve_compute(compute, &ct));
  TRY(check_align({g, nu, params, updates, nu_out, params_out}));
  if (tree->numel == 0) return OPT_OK;
  if (!g) return fail(OPT_EINVAL, "g is NULL");
  Reduce r;
  TRY(setup_reduce(tree, nullptr, nullptr, ext->lr_leaf, nullptr, 0, &r));
  StepArgs<3, 3> a{};
  a.in[0] = g; a.in[1] = nu; a.in[2] = params;
  a.out[0] = updates; a.out[1] = nu_out; a.out[2] = params ? params_out : nullptr;
  a.numel = tree->numel;
  return dispatch<RmsFwdEx, false>(state_dtype, ct, a, r, tree, static_cast<cudaStream_t>(stream),
                                   [&](auto& op) {
                                     fill_rms_fwd(op.base, hp);
                                     fill_ext(op, ext, false);
                                   });
}

int opt_rmsprop_bwd_ex(const opt_tree* tree, const opt_rmsprop_hp* hp, const opt_ext* ext,
                       int state_dtype, int compute, const float* g, const void* nu,
                       const float* params, const float* d_updates, const float* d_nu_out,
                       float* d_g, float* d_nu, float* d_params, double* d_hp, double* d_hp_leaf,
                       void* workspace, size_t workspace_bytes, void* stream) {
  g_err.clear();
  int ct = 0;
  TRY(check_tree(tree));
  TRY(check_rms(hp));
  TRY(check_ext(ext, params, tree));
  TRY(check_state_dtype(state_dtype));
  TRY(resolve_compute(compute, &ct));
  TRY(check_align({g, nu, params, d_updates, d_nu_out, d_g, d_nu, d_params}));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (tree->numel == 0) return zero_outputs(tree, 4, d_hp, d_hp_leaf, s);
  if (!g) return fail(OPT_EINVAL, "g is NULL");
  Reduce r;
  TRY(setup_reduce(tree, d_hp, d_hp_leaf, ext->lr_leaf, workspace, workspace_bytes, &r));
  StepArgs<5, 3> a{};
  a.in[0] = g; a.in[1] = nu; a.in[2] = params; a.in[3] = d_updates; a.in[4] = d_nu_out;
  a.out[0] = d_g; a.out[1] = d_nu; a.out[2] = d_params;
  a.numel = tree->numel;
  return dispatch<RmsBwdEx, true>(state_dtype, ct, a, r, tree, s, [&](auto& op) {
    fill_rms_bwd(op.base, hp);
    fill_ext(op, ext, false);
  });
}

// ------------------------------ fused inner-loss glue (NEXT-2, C3 sweep)
int opt_adam_quad_fwd(const opt_tree* tree, int64_t step, const opt_adam_hp* hp, int state_dtype,
                      int compute, const float* a, const float* phi, const float* theta,
                      const void* mu, const void* nu, float* g_out, void* mu_out, void* nu_out,
                      float* theta_out, void* stream) {
  g_err.clear();
  int ct = 0;
  TRY(check_tree(tree));
  TRY(check_adam(step, hp));
  TRY(check_state_dtype(state_dtype));
  TRY(resolve_compute(compute, &ct));
  TRY(check_align({a, phi, theta, mu, nu, g_out, mu_out, nu_out, theta_out}));
  if (tree->numel == 0) return OPT_OK;
  if (!a || !phi || !theta || !theta_out) return fail(OPT_EINVAL, "a, phi, theta, theta_out required");
  StepArgs<5, 4> x{};
  x.in[0] = a; x.in[1] = theta; x.in[2] = phi; x.in[3] = mu; x.in[4] = nu;
  x.out[0] = g_out; x.out[1] = mu_out; x.out[2] = nu_out; x.out[3] = theta_out;
  x.numel = tree->numel;
  return dispatch<AdamQuadFwd, false>(state_dtype, ct, x, Reduce{}, tree,
                                      static_cast<cudaStream_t>(stream),
                                      [&](auto& op) { fill_adam_fwd(op.base, step, hp); });
}

int opt_adam_quad_rev(const opt_tree* tree, int64_t step, const opt_adam_hp* hp, int state_dtype,
                      int compute, const float* a, const float* g, const void* mu, const void* nu,
                      float* theta_bar, const float* d_mu_out, const float* d_nu_out, float* d_mu,
                      float* d_nu, float* phi_bar, int init_phi, double* d_hp, void* workspace,
                      size_t workspace_bytes, void* stream) {
  g_err.clear();
  int ct = 0;
  TRY(check_tree(tree));
  TRY(check_adam(step, hp));
  TRY(check_state_dtype(state_dtype));
  TRY(resolve_compute(compute, &ct));
  TRY(check_align({a, g, mu, nu, theta_bar, d_mu_out, d_nu_out, d_mu, d_nu, phi_bar}));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (tree->numel == 0) return zero_outputs(tree, 4, d_hp, nullptr, s);
  if (!a || !g || !theta_bar || !phi_bar) return fail(OPT_EINVAL, "a, g, theta_bar, phi_bar required");
  Reduce r;
  TRY(setup_reduce(tree, d_hp, nullptr, nullptr, workspace, workspace_bytes, &r));
  StepArgs<8, 4> x{};
  x.in[0] = a; x.in[1] = g; x.in[2] = mu; x.in[3] = nu; x.in[4] = theta_bar;
  x.in[5] = d_mu_out; x.in[6] = d_nu_out; x.in[7] = init_phi ? nullptr : phi_bar;
  x.out[0] = d_mu; x.out[1] = d_nu; x.out[2] = theta_bar; x.out[3] = phi_bar;
  x.numel = tree->numel;
  return dispatch<AdamQuadRev, true>(state_dtype, ct, x, r, tree, s,
                                     [&](auto& op) { fill_adam_bwd(op.base, step, hp); });
}

// ------------------------------------- RMSProp centred / momentum (NEXT-1)
int opt_rmsprop_cm_fwd(const opt_tree* tree, const opt_rmsprop_cm_hp* hp, const opt_ext* ext,
                       int state_dtype, int compute, const float* g, const void* nu,
                       const void* gavg, const void* buf, const float* params, float* updates,
                       void* nu_out, void* gavg_out, void* buf_out, float* params_out,
                       void* stream) {
  g_err.clear();
  int ct = 0;
  TRY(check_tree(tree));
  TRY(check_rms_cm(hp));
  TRY(check_ext(ext, params, tree));
  TRY(check_state_dtype(state_dtype));
  TRY(resolve_compute(compute, &ct));
  TRY(check_align({g, nu, gavg, buf, params, updates, nu_out, gavg_out, buf_out, params_out}));
  if (tree->numel == 0) return OPT_OK;
  if (!g) return fail(OPT_EINVAL, "g is NULL");
  Reduce r;
  TRY(setup_reduce(tree, nullptr, nullptr, ext->lr_leaf, nullptr, 0, &r));
  StepArgs<5, 5> a{};
  a.in[0] = g; a.in[1] = nu; a.in[2] = hp->centered ? gavg : nullptr; a.in[3] = buf;
  a.in[4] = params;
  a.out[0] = updates; a.out[1] = nu_out; a.out[2] = hp->centered ? gavg_out : nullptr;
  a.out[3] = buf_out; a.out[4] = params ? params_out : nullptr;
  a.numel = tree->numel;
  return dispatch<RmsCmFwd, false>(state_dtype, ct, a, r, tree, static_cast<cudaStream_t>(stream),
                                   [&](auto& op) { fill_rms_cm(op, hp, ext); });
}

int opt_rmsprop_cm_bwd(const opt_tree* tree, const opt_rmsprop_cm_hp* hp, const opt_ext* ext,
                       int state_dtype, int compute, const float* g, const void* nu,
                       const void* gavg, const void* buf, const float* params,
                       const float* d_updates, const float* d_nu_out, const float* d_gavg_out,
                       const float* d_buf_out, float* d_g, float* d_nu, float* d_gavg,
                       float* d_buf, float* d_params, double* d_hp, double* d_hp_leaf,
                       void* workspace, size_t workspace_bytes, void* stream) {
  g_err.clear();
  int ct = 0;
  TRY(check_tree(tree));
  TRY(check_rms_cm(hp));
  TRY(check_ext(ext, params, tree));
  TRY(check_state_dtype(state_dtype));
  TRY(resolve_compute(compute, &ct));
  TRY(check_align({g, nu, gavg, buf, params, d_updates, d_nu_out, d_gavg_out, d_buf_out, d_g,
                   d_nu, d_gavg, d_buf, d_params}));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (tree->numel == 0) return zero_outputs(tree, 5, d_hp, d_hp_leaf, s);
  if (!g) return fail(OPT_EINVAL, "g is NULL");
  Reduce r;
  TRY(setup_reduce(tree, d_hp, d_hp_leaf, ext->lr_leaf, workspace, workspace_bytes, &r));
  StepArgs<9, 5> a{};
  a.in[0] = g; a.in[1] = nu; a.in[2] = hp->centered ? gavg : nullptr; a.in[3] = buf;
  a.in[4] = params; a.in[5] = d_updates; a.in[6] = d_nu_out; a.in[7] = d_gavg_out;
  a.in[8] = d_buf_out;
  a.out[0] = d_g; a.out[1] = d_nu; a.out[2] = d_gavg; a.out[3] = d_buf; a.out[4] = d_params;
  a.numel = tree->numel;
  return dispatch<RmsCmBwd, true>(state_dtype, ct, a, r, tree, s,
                                  [&](auto& op) { fill_rms_cm(op, hp, ext); });
}

// ------------------------------------------------------------------- SGD
int opt_sgd_fwd(const opt_tree* tree, const opt_sgd_hp* hp, int state_dtype, int compute,
                const float* g, const void* mom, float* updates, void* mom_out,
                const float* params, float* params_out, void* stream) {
  g_err.clear();
  int ct = 0;
  TRY(check_tree(tree));
  TRY(check_sgd(hp));
  TRY(check_state_dtype(state_dtype));
  TRY(resolve_compute(compute, &ct));
  TRY(check_align({g, mom, updates, mom_out, params, params_out}));
  if (tree->numel == 0) return OPT_OK;
  if (!g) return fail(OPT_EINVAL, "g is NULL");
  StepArgs<3, 3> a{};
  a.in[0] = g; a.in[1] = mom; a.in[2] = (params && params_out) ? params : nullptr;
  a.out[0] = updates; a.out[1] = mom_out; a.out[2] = (params && params_out) ? params_out : nullptr;
  a.numel = tree->numel;
  return dispatch<SgdFwd, false>(state_dtype, ct, a, Reduce{}, tree,
                                 static_cast<cudaStream_t>(stream),
                                 [&](auto& op) { fill_sgd(op, hp); });
}

int opt_sgd_bwd(const opt_tree* tree, const opt_sgd_hp* hp, int state_dtype, int compute,
                const float* g, const void* mom, const float* d_updates, const float* d_mom_out,
                float* d_g, float* d_mom, double* d_hp, double* d_hp_leaf, void* workspace,
                size_t workspace_bytes, void* stream) {
  g_err.clear();
  int ct = 0;
  TRY(check_tree(tree));
  TRY(check_sgd(hp));
  TRY(check_state_dtype(state_dtype));
  TRY(resolve_compute(compute, &ct));
  TRY(check_align({g, mom, d_updates, d_mom_out, d_g, d_mom}));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (tree->numel == 0) return zero_outputs(tree, 2, d_hp, d_hp_leaf, s);
  if (!g) return fail(OPT_EINVAL, "g is NULL");
  Reduce r;
  TRY(setup_reduce(tree, d_hp, d_hp_leaf, nullptr, workspace, workspace_bytes, &r));
  StepArgs<4, 2> a{};
  a.in[0] = g; a.in[1] = mom; a.in[2] = d_updates; a.in[3] = d_mom_out;
  a.out[0] = d_g; a.out[1] = d_mom;
  a.numel = tree->numel;
  return dispatch<SgdBwd, true>(state_dtype, ct, a, r, tree, s, [&](auto& op) { fill_sgd(op, hp); });
}

int opt_sgd_fwd_ex(const opt_tree* tree, const opt_sgd_hp* hp, const opt_ext* ext,
                   int state_dtype, int compute, const float* g, const void* mom,
                   const float* params, float* updates, void* mom_out, float* params_out,
                   void* stream) {
  g_err.clear();
  int ct = 0;
  TRY(check_tree(tree));
  TRY(check_sgd(hp));
  TRY(check_ext(ext, params, tree));
  TRY(check_state_dtype(state_dtype));
  TRY(resolve_compute(compute, &ct));
  TRY(check_align({g, mom, params, updates, mom_out, params_out}));
  if (tree->numel == 0) return OPT_OK;
  if (!g) return fail(OPT_EINVAL, "g is NULL");
  Reduce r;
  TRY(setup_reduce(tree, nullptr, nullptr, ext->lr_leaf, nullptr, 0, &r));
  StepArgs<3, 3> a{};
  a.in[0] = g; a.in[1] = mom; a.in[2] = params;
  a.out[0] = updates; a.out[1] = mom_out; a.out[2] = params ? params_out : nullptr;
  a.numel = tree->numel;
  return dispatch<SgdFwdEx, false>(state_dtype, ct, a, r, tree, static_cast<cudaStream_t>(stream),
                                   [&](auto& op) {
                                     fill_sgd(op.base, hp);
                                     fill_ext(op, ext, false);
                                   });
}

int opt_sgd_bwd_ex(const opt_tree* tree, const opt_sgd_hp* hp, const opt_ext* ext,
                   int state_dtype, int compute, const float* g, const void* mom,
                   const float* params, const float* d_updates, const float* d_mom_out,
                   float* d_g, float* d_mom, float* d_params, double* d_hp, double* d_hp_leaf,
                   void* workspace, size_t workspace_bytes, void* stream) {
  g_err.clear();
  int ct = 0;
  TRY(check_tree(tree));
  TRY(check_sgd(hp));
  TRY(check_ext(ext, params, tree));
  TRY(check_state_dtype(state_dtype));
  TRY(resolve_compute(compute, &ct));
  TRY(check_align({g, mom, params, d_updates, d_mom_out, d_g, d_mom, d_params}));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (tree->numel == 0) return zero_outputs(tree, 3, d_hp, d_hp_leaf, s);
  if (!g) return fail(OPT_EINVAL, "g is NULL");
  Reduce r;
  TRY(setup_reduce(tree, d_hp, d_hp_leaf, ext->lr_leaf, workspace, workspace_bytes, &r));
  StepArgs<5, 3> a{};
  a.in[0] = g; a.in[1] = mom; a.in[2] = params; a.in[3] = d_updates; a.in[4] = d_mom_out;
  a.out[0] = d_g; a.out[1] = d_mom; a.out[2] = d_params;
  a.numel = tree->numel;
  return dispatch<SgdBwdEx, true>(state_dtype, ct, a, r, tree, s, [&](auto& op) {
    fill_sgd(op.base, hp);
    fill_ext(op, ext, false);
  });
}

// -------------------------------------------------------- misc / glue
const char* opt_status_string(int status) {
  switch (status) {
    case OPT_OK: return "OPT_OK";
    case OPT_EINVAL: return "OPT_EINVAL: invalid argument";
    case OPT_EALIGN: return "OPT_EALIGN: pointer not 16-byte aligned";
    case OPT_ECUDA: return "OPT_ECUDA: CUDA error";
    case OPT_EWORKSPACE: return "OPT_EWORKSPACE: workspace too small";
    default: return "unknown opt_status";
  }
}

const char* opt_last_error(void) { return g_err.c_str(); }
int opt_abi_version(void) { return DIFFOPT_ABI_VERSION; }
int64_t opt_launch_count(void) { return g_launches.load(); }

}  // extern "C"

// ------------------------------------------------------ glue kernels
// apply_updates (row a8) and the synthetic quadratic inner loss of row a9.
namespace {

__global__ void __launch_bounds__(kBlock) apply_kernel(int64_t n, const float* __restrict__ p,
                                                       const float* __restrict__ u,
                                                       float* out) {
  const int64_t nvec = n >> 2, stride = (int64_t)gridDim.x * kBlock;
  for (int64_t v = (int64_t)blockIdx.x * kBlock + threadIdx.x; v < nvec; v += stride) {
    float a[4], b[4];
    load4(p, v, a);
    load4(u, v, b);
    const float o[4] = {a[0] + b[0], a[1] + b[1], a[2] + b[2], a[3] + b[3]};
    store4(out, v, o);
  }
  const int64_t i = (nvec << 2) + threadIdx.x;
  if (blockIdx.x == gridDim.x - 1 && i < n) out[i] = p[i] + u[i];
}

__global__ void __launch_bounds__(kBlock) quad_grad_kernel(int64_t n, const float* __restrict__ a,
                                                           const float* __restrict__ th,
                                                           const float* __restrict__ phi,
                                                           float* g) {
  const int64_t nvec = n >> 2, stride = (int64_t)gridDim.x * kBlock;
  for (int64_t v = (int64_t)blockIdx.x * kBlock + threadIdx.x; v < nvec; v += stride) {
    float x[4], t[4], p[4];
    load4(a, v, x);
    load4(th, v, t);
    load4(phi, v, p);
    const float o[4] = {x[0] * (t[0] - p[0]), x[1] * (t[1] - p[1]), x[2] * (t[2] - p[2]),
                        x[3] * (t[3] - p[3])};
    store4(g, v, o);
  }
  const int64_t i = (nvec << 2) + threadIdx.x;
  if (blockIdx.x == gridDim.x - 1 && i < n) g[i] = a[i] * (th[i] - phi[i]);
}

__global__ void __launch_bounds__(kBlock) quad_rev_kernel(int64_t n, const float* __restrict__ a,
                                                          const float* __restrict__ gb,
                                                          float* thb, float* phib, int init) {
  const int64_t nvec = n >> 2, stride = (int64_t)gridDim.x * kBlock;
  for (int64_t v = (int64_t)blockIdx.x * kBlock + threadIdx.x; v < nvec; v += stride) {
    float x[4], g[4], t[4], p[4];
    load4(a, v, x);
    load4(gb, v, g);
    load4(thb, v, t);
    if (init) {
      p[0] = p[1] = p[2] = p[3] = 0.f;
    } else {
      load4(phib, v, p);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float ag = x[e] * g[e];
      t[e] += ag;
      p[e] -= ag;
    }
    store4(thb, v, t);
    store4(phib, v, p);
  }
  const int64_t i = (nvec << 2) + threadIdx.x;
  if (blockIdx.x == gridDim.x - 1 && i < n) {
    const float ag = a[i] * gb[i];
    thb[i] += ag;
    phib[i] = (init ? 0.f : phib[i]) - ag;
  }
}

template <class K>
int glue_launch(K kernel, int64_t n, cudaStream_t s, int* grid) {
  // elementwise, no partials: one block per 256 vectors (blocks end evenly;
  // see the forward step kernels)
  (void)kernel;
  (void)s;
  const int64_t g = ((n >> 2) + kBlock - 1) / kBlock + 1;
  *grid = (int)(g < 0x7FFFFFFF ? g : 0x7FFFFFFF);
  return OPT_OK;
}

}  // namespace

extern "C" {

int opt_apply_updates(int64_t numel, const float* params, const float* updates, float* out,
                      void* stream) {
  g_err.clear();
  if (numel < 0) return fail(OPT_EINVAL, "numel < 0");
  TRY(check_align({params, updates, out}));
  if (numel == 0) return OPT_OK;
  if (!params || !updates || !out) return fail(OPT_EINVAL, "NULL array");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int grid = 0;
  TRY(glue_launch(apply_kernel, numel, s, &grid));
  apply_kernel<<<grid, kBlock, 0, s>>>(numel, params, updates, out);
  return launched(s);
}

// Fixed-order column sums of a row-major fp64 matrix: one warp per column,
// lane l sums rows l, l+32, ... in order, then a fixed xor-shuffle tree.
__global__ void __launch_bounds__(kBlock) sum_rows_kernel(int64_t rows, int64_t cols,
                                                          const double* __restrict__ in,
                                                          double* __restrict__ out) {
  const int64_t c = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (c >= cols) return;
  double s = 0.0;
  for (int64_t r = lane; r < rows; r += 32) s += in[r * cols + c];
  s = warp_sum(s);
  if (lane == 0) out[c] = s;
}

int opt_sum_rows(int64_t rows, int64_t cols, const double* in, double* out, void* stream) {
  g_err.clear();
  if (rows < 0 || cols < 0) return fail(OPT_EINVAL, "rows = %lld, cols = %lld",
                                        (long long)rows, (long long)cols);
  if (cols == 0) return OPT_OK;
  if (!out) return fail(OPT_EINVAL, "out is NULL");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (rows == 0) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double) * cols, s);
    if (e != cudaSuccess) return fail(OPT_ECUDA, "memset: %s", cudaGetErrorString(e));
    return OPT_OK;
  }
  if (!in) return fail(OPT_EINVAL, "in is NULL");
  const int64_t grid = (cols + kWarps - 1) / kWarps;
  if (grid > 0x7FFFFFFF) return fail(OPT_EINVAL, "too many columns");
  sum_rows_kernel<<<(int)grid, kBlock, 0, s>>>(rows, cols, in, out);
  return launched(s);
}

int opt_copy_rows(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width_bytes,
                  size_t rows, void* stream) {
  g_err.clear();
  if (rows == 0 || width_bytes == 0) return OPT_OK;
  if (!dst || !src) return fail(OPT_EINVAL, "NULL pointer");
  if (rows > 1 && (width_bytes > dpitch || width_bytes > spitch))
    return fail(OPT_EINVAL, "width %zu exceeds a pitch (%zu, %zu)", width_bytes, dpitch, spitch);
  if (rows == 1) dpitch = spitch = width_bytes;
  cudaError_t e = cudaMemcpy2DAsync(dst, dpitch, src, spitch, width_bytes, rows, cudaMemcpyDefault,
                                    static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(OPT_ECUDA, "cudaMemcpy2DAsync: %s", cudaGetErrorString(e));
  return OPT_OK;
}

int opt_quadratic_grad(int64_t numel, const float* a, const float* theta, const float* phi,
                       float* g, void* stream) {
  g_err.clear();
  if (numel < 0) return fail(OPT_EINVAL, "numel < 0");
  TRY(check_align({a, theta, phi, g}));
  if (numel == 0) return OPT_OK;
  if (!a || !theta || !phi || !g) return fail(OPT_EINVAL, "NULL array");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int grid = 0;
  TRY(glue_launch(quad_grad_kernel, numel, s, &grid));
  quad_grad_kernel<<<grid, kBlock, 0, s>>>(numel, a, theta, phi, g);
  return launched(s);
}

int opt_quadratic_rev(int64_t numel, const float* a, const float* g_bar, float* theta_bar,
                      float* phi_bar, int init_phi, void* stream) {
  g_err.clear();
  if (numel < 0) return fail(OPT_EINVAL, "numel < 0");
  TRY(check_align({a, g_bar, theta_bar, phi_bar}));
  if (numel == 0) return OPT_OK;
  if (!a || !g_bar || !theta_bar || !phi_bar) return fail(OPT_EINVAL, "NULL array");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int grid = 0;
  TRY(glue_launch(quad_rev_kernel, numel, s, &grid));
  quad_rev_kernel<<<grid, kBlock, 0, s>>>(numel, a, g_bar, theta_bar, phi_bar, init_phi);
  return launched(s);
}

}  // extern "C"

// ------------------------------------------- zero-order ES (NEXT-3, es.cuh)

// ------------------------------------------ sharded Adam step over peer memory
namespace dopt {
struct PeerArgs {
  const float* g[OPT_MAX_PEERS];
  float* p[OPT_MAX_PEERS];
};

// One pass over the shard: W peer gradient loads (summed in rank order, so
// every rank computes bit-identical sums), the Adam step on the local state,
// and W peer parameter stores: reduce-scatter + step + all-gather fused.
__global__ void __launch_bounds__(256) adam_peers_kernel(int world, PeerArgs pa, int64_t lo,
                                                         int64_t nvec, int64_t tail, float scale,
                                                         AdamFwd<float> op, float* __restrict__ mu,
                                                         float* __restrict__ nu,
                                                         const float* __restrict__ params) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec + tail; v += stride) {
    const bool vec = v < nvec;
    const int64_t i0 = vec ? 4 * v : 4 * nvec + (v - nvec);  // shard index
    const int nl = vec ? 4 : 1;
    float g[4] = {0.f, 0.f, 0.f, 0.f};
    for (int w = 0; w < world; ++w) {
      if (vec) {
        const float4 x = __ldcv(reinterpret_cast<const float4*>(pa.g[w] + lo + i0));
        g[0] += x.x, g[1] += x.y, g[2] += x.z, g[3] += x.w;
      } else {
        g[0] += __ldcv(pa.g[w] + lo + i0);
      }
    }
    float m[4], vv[4], th[4], out[4];
    for (int k = 0; k < nl; ++k) {
      m[k] = mu[i0 + k], vv[k] = nu[i0 + k], th[k] = params[lo + i0 + k];
      float u, m1, v1;
      op.apply(g[k] * scale, m[k], vv[k], u, m1, v1);
      mu[i0 + k] = m1, nu[i0 + k] = v1;
      out[k] = th[k] + u;
    }
    for (int w = 0; w < world; ++w) {
      if (vec)
        __stcg(reinterpret_cast<float4*>(pa.p[w] + lo + i0), make_float4(out[0], out[1], out[2], out[3]));
      else
        __stcg(pa.p[w] + lo + i0, out[0]);
    }
  }
}
}  // namespace dopt

extern "C" int opt_adam_fwd_peers(int world, const opt_peers* peers, int64_t lo, int64_t n_shard,
                                  int64_t step, const opt_adam_hp* hp, double grad_scale,
                                  float* mu, float* nu, const float* params, void* stream) {
  using namespace dopt;
  g_err.clear();
  TRY(check_adam(step, hp));
  if (world < 1 || world > OPT_MAX_PEERS) return fail(OPT_EINVAL, "world = %d", world);
  if (!peers) return fail(OPT_EINVAL, "peers is NULL");
  if (lo < 0 || n_shard < 0) return fail(OPT_EINVAL, "bad shard range");
  if (lo % 4) return fail(OPT_EALIGN, "lo = %lld is not a multiple of 4", (long long)lo);
  if (!(grad_scale == grad_scale)) return fail(OPT_EINVAL, "grad_scale is NaN");
  if (n_shard == 0) return OPT_OK;
  if (!mu || !nu || !params) return fail(OPT_EINVAL, "mu / nu / params is NULL");
  TRY(check_align({mu, nu, params}));
  PeerArgs pa{};
  for (int w = 0; w < world; ++w) {
    if (!peers->g[w] || !peers->params[w]) return fail(OPT_EINVAL, "peer %d pointer is NULL", w);
    TRY(check_align({peers->g[w], peers->params[w]}));
    pa.g[w] = peers->g[w], pa.p[w] = peers->params[w];
  }
  AdamFwd<float> op;
  fill_adam_fwd(op, step, hp);
  const int64_t nvec = n_shard / 4, tail = n_shard - 4 * nvec;
  int64_t blocks = (nvec + tail + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  adam_peers_kernel<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      world, pa, lo, nvec, tail, (float)grad_scale, op, mu, nu, params);
  return launched(static_cast<cudaStream_t>(stream));
}

// ------------------------------------------ device-side peer barrier (flags)
namespace dopt {
struct PeerFlags {
  unsigned long long* f[OPT_MAX_PEERS];
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// One warp: lane w < world publishes `epoch` into rank `rank`'s slot of
// peer w's flag array (after a system-scope fence, so every write this
// rank's stream issued before -- its gradient, or its parameter stores into
// every peer -- is visible first), then lane w spins (acquire loads, backed
// off) until peer w's slot in this rank's own array reaches `epoch`. A wait
// longer than timeout_ns writes 1 to *status and gives up (no hang).
__global__ void peer_signal_wait_kernel(int world, int rank, int slot, PeerFlags pf,
                                        unsigned long long epoch, unsigned long long timeout_ns,
                                        int* status) {
  const int w = threadIdx.x;
  __threadfence_system();
  __syncwarp();
  if (w < world) st_release_sys(pf.f[w] + (int64_t)slot * OPT_MAX_PEERS + rank, epoch);
  if (w < world) {
    const unsigned long long* mine = pf.f[rank] + (int64_t)slot * OPT_MAX_PEERS + w;
    const unsigned long long t0 = globaltimer();
    unsigned ns = 32;
    while (ld_acquire_sys(mine) < epoch) {
      if (globaltimer() - t0 > timeout_ns) {
        atomicExch(status, 1);
        break;
      }
      __nanosleep(ns);
      if (ns < 1024) ns <<= 1;
    }
  }
  __syncwarp();
  __threadfence_system();
}
}  // namespace dopt

extern "C" int opt_peer_signal_wait(int world, int rank, int slot, const opt_peer_flags* flags,
                                    uint64_t epoch, double timeout_s, int* status, void* stream) {
  using namespace dopt;
  g_err.clear();
  if (world < 1 || world > OPT_MAX_PEERS) return fail(OPT_EINVAL, "world = %d", world);
  if (rank < 0 || rank >= world) return fail(OPT_EINVAL, "rank = %d", rank);
  if (slot < 0 || slot > 1) return fail(OPT_EINVAL, "slot = %d (0 = ready, 1 = done)", slot);
  if (!flags || !status) return fail(OPT_EINVAL, "flags / status is NULL");
  if (epoch == 0) return fail(OPT_EINVAL, "epoch must be >= 1 (flags start at 0)");
  if (!(timeout_s > 0.0)) return fail(OPT_EINVAL, "timeout must be > 0");
  PeerFlags pf{};
  for (int w = 0; w < world; ++w) {
    if (!flags->f[w]) return fail(OPT_EINVAL, "flags of peer %d is NULL", w);
    if ((uintptr_t)flags->f[w] & 7) return fail(OPT_EALIGN, "flags of peer %d not 8-byte aligned", w);
    pf.f[w] = reinterpret_cast<unsigned long long*>(flags->f[w]);
  }
  const double ns = timeout_s * 1e9;
  peer_signal_wait_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
      world, rank, slot, pf, (unsigned long long)epoch,
      ns > 1.8e19 ? 18000000000000000000ull : (unsigned long long)ns, status);
  return launched(static_cast<cudaStream_t>(stream));
}

#include "es.cuh"

extern "C" {

int opt_es_perturb(int64_t numel, int64_t n_samples, int64_t sample0, int antithetic,
                   double sigma, uint64_t seed, const float* theta, float* out, void* stream) {
  g_err.clear();
  if (numel < 0 || n_samples < 0 || sample0 < 0) return fail(OPT_EINVAL, "negative size");
  if (n_samples > kEsMaxSamples)
    return fail(OPT_EINVAL, "n_samples = %lld > %d per call (use sample0 chunks)",
                (long long)n_samples, kEsMaxSamples);
  if (!(std::isfinite(sigma) && sigma > 0)) return fail(OPT_EINVAL, "sigma must be > 0");
  TRY(check_align({theta, out}));
  if (numel == 0 || n_samples == 0) return OPT_OK;
  if (!theta || !out) return fail(OPT_EINVAL, "NULL array");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int sms = 0;
  TRY(sm_count(&sms));
  const int64_t nvec = (numel + 3) >> 2;
  const int64_t capacity = (int64_t)sms * 2048;  // resident threads
  // samples per thread: all of them when the tree alone fills the GPU
  int64_t groups = capacity / (nvec > 0 ? nvec : 1);
  if (groups < 1) groups = 1;
  if (groups > n_samples) groups = n_samples;
  const int64_t spg = (n_samples + groups - 1) / groups;
  const int64_t work = nvec * ((n_samples + spg - 1) / spg);
  int64_t grid = (work + 255) / 256;  // one work item per thread (no persistent cap: as
  if (grid > 0x7FFFFFFF) grid = 0x7FFFFFFF;  // for the forward step kernels, blocks end evenly)
  if (grid < 1) grid = 1;
  const size_t smem = sizeof(uint64_t) * (size_t)n_samples;
  static const cudaError_t attr = cudaFuncSetAttribute(
      es_perturb_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
      (int)(sizeof(uint64_t) * kEsMaxSamples));
  if (attr != cudaSuccess) return fail(OPT_ECUDA, "smem attribute: %s", cudaGetErrorString(attr));
  es_perturb_kernel<<<(int)grid, 256, smem, s>>>(numel, n_samples, sample0, antithetic,
                                                 (float)sigma, seed, spg, theta, out);
  return launched(s);
}

int opt_es_grad(int64_t numel, int64_t n_samples, int antithetic, double sigma, uint64_t seed,
                const float* f_values, float* grad, void* stream) {
  g_err.clear();
  if (numel < 0 || n_samples < 1) return fail(OPT_EINVAL, "numel < 0 or n_samples < 1");
  if (n_samples > kEsMaxSamples)
    return fail(OPT_EINVAL, "n_samples = %lld > %d", (long long)n_samples, kEsMaxSamples);
  if (!(std::isfinite(sigma) && sigma > 0)) return fail(OPT_EINVAL, "sigma must be > 0");
  TRY(check_align({grad}));
  if (numel == 0) return OPT_OK;
  if (!f_values || !grad) return fail(OPT_EINVAL, "NULL array");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int sms = 0;
  TRY(sm_count(&sms));
  const int64_t nvec = (numel + 3) >> 2;
  const bool split = nvec < (int64_t)sms * 512 && n_samples >= 64;  // small tree, many samples
  const int64_t threads = split ? nvec * 32 : nvec;
  int64_t grid = (threads + 255) / 256;
  // every block stages the samples' keys and weights: with few samples a
  // full grid (blocks end evenly) is cheap; with many, stay persistent
  if (n_samples > 256 && grid > (int64_t)sms * 8) grid = (int64_t)sms * 8;
  if (grid > 0x7FFFFFFF) grid = 0x7FFFFFFF;
  if (grid < 1) grid = 1;
  const size_t smem = (sizeof(uint64_t) + sizeof(float)) * (size_t)n_samples;
  const int max_smem = (int)((sizeof(uint64_t) + sizeof(float)) * kEsMaxSamples);
  static const cudaError_t attr0 = cudaFuncSetAttribute(
      es_grad_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem);
  static const cudaError_t attr1 = cudaFuncSetAttribute(
      es_grad_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem);
  if (attr0 != cudaSuccess || attr1 != cudaSuccess)
    return fail(OPT_ECUDA, "smem attribute failed");
  const double scale = antithetic ? 1.0 / (2.0 * (double)n_samples * sigma)
                                  : 1.0 / ((double)n_samples * sigma);
  if (split)
    es_grad_kernel<true><<<(int)grid, 256, smem, s>>>(numel, n_samples, antithetic, scale, seed,
                                                      f_values, grad);
  else
    es_grad_kernel<false><<<(int)grid, 256, smem, s>>>(numel, n_samples, antithetic, scale, seed,
                                                       f_values, grad);
  return launched(s);
}

}  // extern "C"

// ------------------------------------- implicit gradients (NEXT-4, implicit.cuh)
#include "implicit.cuh"

namespace {

template <int MODE>
int cg_launch(int64_t n, float* x, float* r, float* p, const float* Ap, const float* b,
              const float* Ax0, double* state, void* ws, size_t wsb, void* stream) {
  if (n < 0) return fail(OPT_EINVAL, "n < 0");
  TRY(check_align({x, r, p, Ap, b, Ax0}));
  if (!state) return fail(OPT_EINVAL, "state is NULL");
  const bool reduce = MODE != CG_DIR;
  const size_t need = kCounterBytes + sizeof(double) * (size_t)kMaxGrid;
  if (reduce && (!ws || wsb < need))
    return fail(OPT_EWORKSPACE, "workspace %p of %zu bytes; need %zu", ws, wsb, need);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CgArgs a{};
  a.n = n; a.x = x; a.r = r; a.p = p; a.Ap = Ap; a.b = b; a.Ax0 = Ax0; a.state = state;
  if (reduce) {
    a.counter = static_cast<unsigned int*>(ws);
    a.partials = reinterpret_cast<double*>(static_cast<char*>(ws) + kCounterBytes);
  }
  auto k = cg_kernel<MODE>;
  int grid = 0;
  TRY(grid_for(k, ((n >> 2) + kBlock - 1) / kBlock + 1, 0, &grid));
  k<<<grid, kBlock, 0, s>>>(a);
  return launched(s);
}

}  // namespace

extern "C" {

int opt_cg_init(int64_t n, const float* b, const float* Ax0, float* r, float* p, double* state,
                void* workspace, size_t workspace_bytes, void* stream) {
  g_err.clear();
  if (!b || !r || !p) return fail(OPT_EINVAL, "NULL array");
  return cg_launch<CG_INIT>(n, nullptr, r, p, nullptr, b, Ax0, state, workspace,
                            workspace_bytes, stream);
}

int opt_cg_alpha(int64_t n, const float* p, const float* Ap, double* state, void* workspace,
                 size_t workspace_bytes, void* stream) {
  g_err.clear();
  if (!p || !Ap) return fail(OPT_EINVAL, "NULL array");
  return cg_launch<CG_ALPHA_MODE>(n, nullptr, nullptr, const_cast<float*>(p), Ap, nullptr,
                                  nullptr, state, workspace, workspace_bytes, stream);
}

int opt_cg_update(int64_t n, float* x, float* r, const float* p, const float* Ap, double* state,
                  void* workspace, size_t workspace_bytes, void* stream) {
  g_err.clear();
  if (!x || !r || !p || !Ap) return fail(OPT_EINVAL, "NULL array");
  return cg_launch<CG_UPD>(n, x, r, const_cast<float*>(p), Ap, nullptr, nullptr, state,
                           workspace, workspace_bytes, stream);
}

int opt_cg_direction(int64_t n, float* p, const float* r, const double* state, void* stream) {
  g_err.clear();
  if (!p || !r) return fail(OPT_EINVAL, "NULL array");
  return cg_launch<CG_DIR>(n, nullptr, const_cast<float*>(r), p, nullptr, nullptr, nullptr,
                           const_cast<double*>(state), nullptr, 0, stream);
}

int opt_neumann_step(int64_t n, float* v, const float* Av, float* x, double alpha,
                     void* stream) {
  g_err.clear();
  if (n < 0) return fail(OPT_EINVAL, "n < 0");
  if (!std::isfinite(alpha)) return fail(OPT_EINVAL, "alpha not finite");
  TRY(check_align({v, Av, x}));
  if (n == 0) return OPT_OK;
  if (!v || !Av || !x) return fail(OPT_EINVAL, "NULL array");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int grid = 0;
  TRY(glue_launch(neumann_kernel, n, s, &grid));
  neumann_kernel<<<grid, kBlock, 0, s>>>(n, v, Av, x, (float)alpha);
  return launched(s);
}

}  // extern "C"
