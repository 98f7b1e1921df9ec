// step_kernel.cuh -- the one-pass multi-tensor kernel shared by all six ops.
//
// Design:
//   * The tensor tree is one flat buffer per role, so the elementwise math
//     never looks at leaf boundaries: a persistent grid (148 SMs x resident
//     blocks) grid-strides over 4-element vectors, U vectors per thread per
//     iteration with all loads issued before any math (memory-level
//     parallelism), streaming (.cs) 16-byte loads/stores, one HBM pass.
//   * Hyper-gradient sums (Op::NH > 0): per-thread fp64 accumulators ->
//     warp xor-shuffle -> shared memory -> one fp64 partial per block in the
//     workspace -> the last block to arrive (atomic ticket + threadfence)
//     sums the partials in block order. One launch, no atomics on data, and
//     bitwise reproducible for a fixed grid (reading Z12).
//   * Per-leaf sums (d_hp_leaf): the offset table is staged in shared memory
//     and split into leaf-aligned tiles of kTile elements (a scan of
//     ceil(len/kTile) per leaf, done by every block); each tile's partial goes
//     to the workspace and the last block sums every leaf's tiles in order.
#pragma once
#include <stdint.h>

#include "ops.cuh"
#include "vec.cuh"

namespace dopt {

constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;
constexpr int64_t kTile = 1024;      // leaf-mode tile (elements), one warp each
constexpr int kMaxLeafSmem = 4096;   // leaf-mode limit on n_leaves (smem table)

template <int NIN, int NOUT>
struct StepArgs {
  const void* in[NIN];
  void* out[NOUT];
  int64_t numel;
  double* d_hp;          // [NH] final sums (may be NULL)
  double* d_hp_leaf;     // [n_leaves][NH] (leaf mode)
  double* partials;      // workspace: per block (uniform) or per tile (leaf)
  unsigned int* counter; // workspace: arrival ticket, left at 0
  const int64_t* offsets;  // device offsets (leaf mode)
  const float* lr_leaf;    // per-leaf learning rates (leaf mode) or NULL
  int64_t* tile_prefix;    // workspace (leaf mode): first tile of every leaf, [n_leaves+1]
  int64_t n_leaves;
  int64_t n_tiles;
  int want_hp;
};

// ------------------------------------------------------------ element IO
template <class Op, class ST>
__device__ __forceinline__ void load_vec(const StepArgs<Op::NIN, Op::NOUT>& a, int64_t v,
                                         float (&x)[Op::NIN][4]) {
#pragma unroll
  for (int i = 0; i < Op::NIN; ++i) {
    if (a.in[i]) {
      if (Op::in_state(i))
        load4(static_cast<const ST*>(a.in[i]), v, x[i]);
      else
        load4(static_cast<const float*>(a.in[i]), v, x[i]);
    } else {
      x[i][0] = x[i][1] = x[i][2] = x[i][3] = 0.f;
    }
  }
}

template <class Op, class ST>
__device__ __forceinline__ void compute_store_vec(const Op& op,
                                                  const StepArgs<Op::NIN, Op::NOUT>& a,
                                                  int64_t v, const float (&x)[Op::NIN][4],
                                                  double* acc, bool want_hp) {
  typedef typename Op::CT CT;
  constexpr int NH = Op::NH > 0 ? Op::NH : 1;
  CT y[Op::NOUT][4];
  CT hv[NH];  // this vector's hyper terms in CT, then one fp64 add each
#pragma unroll
  for (int k = 0; k < NH; ++k) hv[k] = CT(0);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    float xe[Op::NIN];
#pragma unroll
    for (int i = 0; i < Op::NIN; ++i) xe[i] = x[i][e];
    CT ye[Op::NOUT];
    op(xe, ye, hv, want_hp);
#pragma unroll
    for (int o = 0; o < Op::NOUT; ++o) y[o][e] = ye[o];
  }
  if (Op::NH > 0 && want_hp) {
#pragma unroll
    for (int k = 0; k < Op::NH; ++k) acc[k] += (double)hv[k];
  }
#pragma unroll
  for (int o = 0; o < Op::NOUT; ++o) {
    if (a.out[o]) {
      if (Op::out_state(o))
        store4c(static_cast<ST*>(a.out[o]), v, y[o]);
      else
        store4c(static_cast<float*>(a.out[o]), v, y[o]);
    }
  }
}

template <class Op, class ST>
__device__ __forceinline__ void process_elem(const Op& op, const StepArgs<Op::NIN, Op::NOUT>& a,
                                             int64_t i, double* acc, bool want_hp) {
  typedef typename Op::CT CT;
  float xe[Op::NIN];
#pragma unroll
  for (int k = 0; k < Op::NIN; ++k) {
    if (a.in[k])
      xe[k] = Op::in_state(k) ? load1(static_cast<const ST*>(a.in[k]), i)
                              : load1(static_cast<const float*>(a.in[k]), i);
    else
      xe[k] = 0.f;
  }
  CT ye[Op::NOUT];
  constexpr int NH = Op::NH > 0 ? Op::NH : 1;
  CT hv[NH];
#pragma unroll
  for (int k = 0; k < NH; ++k) hv[k] = CT(0);
  op(xe, ye, hv, want_hp);
  if (Op::NH > 0 && want_hp) {
#pragma unroll
    for (int k = 0; k < Op::NH; ++k) acc[k] += (double)hv[k];
  }
#pragma unroll
  for (int o = 0; o < Op::NOUT; ++o) {
    if (a.out[o]) {
      if (Op::out_state(o))
        store1(static_cast<ST*>(a.out[o]), i, ye[o]);
      else
        store1(static_cast<float*>(a.out[o]), i, ye[o]);
    }
  }
}

// Vectors [v0, v1) handled by `nthreads` threads (this one is `tid`), U
// vectors in flight per thread.
template <class Op, class ST, int U>
__device__ __forceinline__ void process_vectors(const Op& op,
                                                const StepArgs<Op::NIN, Op::NOUT>& a,
                                                int64_t v0, int64_t v1, int64_t tid,
                                                int64_t nthreads, double* acc, bool want_hp) {
  int64_t v = v0 + tid;
  for (; v + (U - 1) * nthreads < v1; v += U * nthreads) {
    float x[U][Op::NIN][4];
#pragma unroll
    for (int u = 0; u < U; ++u) load_vec<Op, ST>(a, v + u * nthreads, x[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) compute_store_vec<Op, ST>(op, a, v + u * nthreads, x[u], acc, want_hp);
  }
  for (; v < v1; v += nthreads) {
    float x[Op::NIN][4];
    load_vec<Op, ST>(a, v, x);
    compute_store_vec<Op, ST>(op, a, v, x, acc, want_hp);
  }
}

// --------------------------------------------------------- reductions
__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// Block sum of acc[NH]; result valid in thread 0. Fixed order.
template <int NH>
__device__ __forceinline__ void block_sum(double* acc, double (*sm)[kWarps]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NH; ++k) {
    double s = warp_sum(acc[k]);
    if (lane == 0) sm[k][warp] = s;
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < NH; ++k) {
      double s = lane < kWarps ? sm[k][lane] : 0.0;
      acc[k] = warp_sum(s);
    }
  }
  __syncthreads();
}

// Arrival ticket: returns true in every thread of the last block to finish.
__device__ __forceinline__ bool last_block(unsigned int* counter, unsigned int nblocks) {
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned int t = atomicAdd(counter, 1u);
    s_last = (t == nblocks - 1);
  }
  __syncthreads();
  if (s_last) __threadfence();
  return s_last;
}

// PDL hooks (no-ops unless the launch used programmatic serialization).
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ------------------------------------------------------- uniform kernel
template <class Op, class ST, int U, int MINB>
__global__ void __launch_bounds__(kBlock, MINB) step_uniform(const Op op,
                                                       const StepArgs<Op::NIN, Op::NOUT> a) {
  constexpr int NH = Op::NH > 0 ? Op::NH : 1;
  const bool want_hp = Op::NH > 0 && a.want_hp;
  double acc[NH];
#pragma unroll
  for (int k = 0; k < NH; ++k) acc[k] = 0.0;

  const int64_t nvec = a.numel >> 2;
  const int64_t nthreads = (int64_t)gridDim.x * kBlock;
  const int64_t tid = (int64_t)blockIdx.x * kBlock + threadIdx.x;
  pdl_wait();
  process_vectors<Op, ST, U>(op, a, 0, nvec, tid, nthreads, acc, want_hp);
  pdl_trigger();
  // ragged tail (numel % 4 elements) -> the last block
  const int64_t tail0 = nvec << 2;
  if (blockIdx.x == gridDim.x - 1 && tail0 + threadIdx.x < a.numel)
    process_elem<Op, ST>(op, a, tail0 + threadIdx.x, acc, want_hp);

  if constexpr (Op::NH > 0) {
    if (!want_hp) return;  // uniform across the grid
    __shared__ double sm[NH][kWarps];
    block_sum<NH>(acc, sm);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 0; k < NH; ++k) a.partials[(int64_t)blockIdx.x * NH + k] = acc[k];
    }
    if (last_block(a.counter, gridDim.x)) {
      double s[NH];
#pragma unroll
      for (int k = 0; k < NH; ++k) s[k] = 0.0;
      for (int64_t b = threadIdx.x; b < gridDim.x; b += kBlock)
#pragma unroll
        for (int k = 0; k < NH; ++k) s[k] += __ldcg(&a.partials[b * NH + k]);
      block_sum<NH>(s, sm);
      if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < NH; ++k)
          if (a.d_hp) a.d_hp[k] = s[k];
        *a.counter = 0u;
      }
    }
  }
}

// ---------------------------------------------------------- leaf kernel
// Dynamic smem: s_off[n_leaves+1], s_tp[n_leaves+1] (first tile of leaf l).
__device__ __forceinline__ int64_t tiles_of(int64_t len) { return (len + kTile - 1) / kTile; }

template <class Op, class ST, int U, int MINB>
__global__ void __launch_bounds__(kBlock, MINB) step_leaf(const Op op,
                                                    const StepArgs<Op::NIN, Op::NOUT> a) {
  constexpr int NH = Op::NH > 0 ? Op::NH : 1;
  const bool want_hp = Op::NH > 0 && a.want_hp;
  extern __shared__ int64_t s_dyn[];
  int64_t* s_off = s_dyn;
  int64_t* s_tp = s_dyn + (a.n_leaves + 1);
  __shared__ int64_t s_scan[kBlock];

  const int64_t nl = a.n_leaves;
  pdl_wait();
  // stage offsets; per-thread contiguous chunk for the scan
  for (int64_t l = threadIdx.x; l <= nl; l += kBlock) s_off[l] = a.offsets[l];
  __syncthreads();
  const int64_t per = (nl + kBlock - 1) / kBlock;
  const int64_t l0 = threadIdx.x * per, l1 = min(l0 + per, nl);
  int64_t local = 0;
  for (int64_t l = l0; l < l1; ++l) local += tiles_of(s_off[l + 1] - s_off[l]);
  s_scan[threadIdx.x] = local;
  __syncthreads();
  if (threadIdx.x == 0) {  // 256-entry exclusive scan
    int64_t run = 0;
    for (int t = 0; t < kBlock; ++t) {
      int64_t c = s_scan[t];
      s_scan[t] = run;
      run += c;
    }
  }
  __syncthreads();
  {
    int64_t run = s_scan[threadIdx.x];
    for (int64_t l = l0; l < l1; ++l) {
      s_tp[l] = run;
      run += tiles_of(s_off[l + 1] - s_off[l]);
    }
    if (threadIdx.x == kBlock - 1) s_tp[nl] = a.n_tiles;
  }
  __syncthreads();
  if (blockIdx.x == 0 && want_hp)  // for leaf_finalize
    for (int64_t l = threadIdx.x; l <= nl; l += kBlock) a.tile_prefix[l] = s_tp[l];

  // Warp tiles: warp w of the grid takes tiles w, w + nwarps, ...; the tile's
  // hyper sums are reduced with shuffles only (no block barrier in the loop).
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * kWarps;
  for (int64_t tile = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); tile < a.n_tiles;
       tile += nwarps) {
    // leaf = last l with s_tp[l] <= tile and a non-empty range
    int64_t lo = 0, hi = nl - 1;
    while (lo < hi) {
      int64_t mid = (lo + hi + 1) >> 1;
      if (s_tp[mid] <= tile) lo = mid; else hi = mid - 1;
    }
    const int64_t leaf_end = s_off[lo + 1];
    const int64_t start = s_off[lo] + (tile - s_tp[lo]) * kTile;
    const int64_t end = min(start + kTile, leaf_end);
    Op opt = op;  // this tile's leaf learning rate (per-leaf lr variants)
    if (a.lr_leaf) opt.set_lr((typename Op::CT)a.lr_leaf[lo]);
    double acc[NH];
#pragma unroll
    for (int k = 0; k < NH; ++k) acc[k] = 0.0;
    const int64_t va = (start + 3) >> 2, vb = end >> 2;
    if (va < vb) {
      process_vectors<Op, ST, U>(opt, a, va, vb, lane, 32, acc, want_hp);
      if (start + lane < (va << 2)) process_elem<Op, ST>(opt, a, start + lane, acc, want_hp);
      if ((vb << 2) + lane < end) process_elem<Op, ST>(opt, a, (vb << 2) + lane, acc, want_hp);
    } else {
      for (int64_t i = start + lane; i < end; i += 32) process_elem<Op, ST>(opt, a, i, acc, want_hp);
    }
    if (want_hp) {
#pragma unroll
      for (int k = 0; k < NH; ++k) acc[k] = warp_sum(acc[k]);
      if (lane == 0)
#pragma unroll
        for (int k = 0; k < NH; ++k) a.partials[tile * NH + k] = acc[k];
    }
  }
}

// Per-leaf sums of the tile partials (second launch of leaf mode): one warp
// per leaf, lanes stride over the leaf's tiles, xor-shuffle; one fp64 partial
// per block of the leaf sums (in warp = leaf order) and the last block sums
// those in block order into d_hp. Deterministic for a fixed grid.
template <int NH>
__global__ void __launch_bounds__(kBlock) leaf_finalize(const double* partials,
                                                        const int64_t* tile_prefix,
                                                        int64_t n_leaves, double* d_hp_leaf,
                                                        double* d_hp, double* block_part,
                                                        unsigned int* counter) {
  pdl_wait();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t l = (int64_t)blockIdx.x * kWarps + warp;
  double s[NH];
#pragma unroll
  for (int k = 0; k < NH; ++k) s[k] = 0.0;
  if (l < n_leaves) {
    const int64_t t0 = tile_prefix[l], t1 = tile_prefix[l + 1];
    for (int64_t t = t0 + lane; t < t1; t += 32)
#pragma unroll
      for (int k = 0; k < NH; ++k) s[k] += __ldcg(&partials[t * NH + k]);
  }
#pragma unroll
  for (int k = 0; k < NH; ++k) s[k] = warp_sum(s[k]);
  __shared__ double sm[NH][kWarps];
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NH; ++k) {
      if (l < n_leaves && d_hp_leaf) d_hp_leaf[l * NH + k] = s[k];
      sm[k][warp] = l < n_leaves ? s[k] : 0.0;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NH; ++k) {
      double b = 0.0;
      for (int w = 0; w < kWarps; ++w) b += sm[k][w];
      block_part[(int64_t)blockIdx.x * NH + k] = b;
    }
  }
  if (last_block(counter, gridDim.x)) {
    double tot[NH];
#pragma unroll
    for (int k = 0; k < NH; ++k) tot[k] = 0.0;
    for (int64_t b = threadIdx.x; b < gridDim.x; b += kBlock)
#pragma unroll
      for (int k = 0; k < NH; ++k) tot[k] += __ldcg(&block_part[b * NH + k]);
    block_sum<NH>(tot, sm);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 0; k < NH; ++k)
        if (d_hp) d_hp[k] = tot[k];
      *counter = 0u;
    }
  }
}

}  // namespace dopt
