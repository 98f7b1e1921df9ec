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
//   * Per-leaf sums (d_hp_leaf) / per-leaf lr: the same grid-stride over
//     256-element chunks, each chunk split at leaf boundaries (binary search
//     in the shared-memory offset table); one fp64 partial per (chunk, leaf)
//     piece at slot chunk + leaf, then two fixed-order folds (see below).
#pragma once
#include <stdint.h>

#include "ops.cuh"
#include "vec.cuh"

namespace dopt {

#ifndef DOPT_DYN_TAIL_PCT  // percent of the vectors claimed dynamically (0 = off)
#define DOPT_DYN_TAIL_PCT 5
#endif
constexpr int64_t kDynTailPct = DOPT_DYN_TAIL_PCT;
constexpr int64_t kDynTailMinVec = int64_t(1) << 24;  // >= 2^26 elements
constexpr int64_t kMaxParts = 4096;  // partial slots in the workspace (= kMaxGrid)
#ifndef DOPT_SPAN
#define DOPT_SPAN 0
#endif

constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;
constexpr int kChunkShift = 8;                // leaf mode: 256-element chunks, one warp each
constexpr int64_t kChunk = int64_t(1) << kChunkShift;
constexpr int kSuperShift = kChunkShift + 5;  // leaf mode: super-chunks of 32 chunks
constexpr int kMaxLeafSmem = 4096;            // offset table staged in smem up to this

__host__ __device__ constexpr int64_t n_chunks_of(int64_t numel) {
  return (numel + kChunk - 1) >> kChunkShift;
}
__host__ __device__ constexpr int64_t n_supers_of(int64_t numel) {
  return (numel + (int64_t(1) << kSuperShift) - 1) >> kSuperShift;
}

template <int NIN, int NOUT>
struct StepArgs {
  const void* in[NIN];
  void* out[NOUT];
  int64_t numel;
  double* d_hp;          // [NH] final sums (may be NULL)
  double* d_hp_leaf;     // [n_leaves][NH] (leaf mode)
  double* partials;      // workspace: per block (uniform) or per piece slot (leaf)
  unsigned int* counter; // workspace: arrival ticket, left at 0
  const int64_t* offsets;  // device offsets (leaf mode)
  const float* lr_leaf;    // per-leaf learning rates (leaf mode) or NULL
  int64_t n_leaves;
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

// Warp-span variant: each warp takes 32*U CONSECUTIVE vectors per iteration
// (U x 512 B contiguous per array instead of U strided 512 B pieces), grid
// stride over spans; the < 32*U leftover vectors go thread-strided.
template <class Op, class ST, int U>
__device__ __forceinline__ void process_spans(const Op& op, const StepArgs<Op::NIN, Op::NOUT>& a,
                                              int64_t nvec, int64_t tid, int64_t nthreads,
                                              double* acc, bool want_hp) {
  constexpr int64_t SPAN = 32 * U;
  const int64_t lane = tid & 31, gw = tid >> 5, nw = nthreads >> 5;
  const int64_t full = nvec / SPAN * SPAN;
  for (int64_t base = gw * SPAN; base < full; base += nw * SPAN) {
    float x[U][Op::NIN][4];
#pragma unroll
    for (int u = 0; u < U; ++u) load_vec<Op, ST>(a, base + u * 32 + lane, x[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
      compute_store_vec<Op, ST>(op, a, base + u * 32 + lane, x[u], acc, want_hp);
  }
  for (int64_t v = full + tid; v < nvec; v += nthreads) {
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

// This thread's share of the final sum over nparts partial rows (rows
// threadIdx.x, +kBlock, +2 kBlock, ... added in that order): four rows' loads
// are issued before any add, so the last block waits for one L2 round trip
// per four rows instead of one per row (same order, same bits).
template <int NH>
__device__ __forceinline__ void sum_partials(const double* __restrict__ part, int64_t nparts,
                                             double* s) {
  int64_t b = threadIdx.x;
  for (; b + 3 * kBlock < nparts; b += 4 * kBlock) {
    double t[4][NH];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int k = 0; k < NH; ++k) t[u][k] = __ldcg(&part[(b + u * kBlock) * NH + k]);
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int k = 0; k < NH; ++k) s[k] += t[u][k];
  }
  double t[3][NH];
  int r = 0;
#pragma unroll
  for (int u = 0; u < 3; ++u)
    if (b + u * kBlock < nparts) {
#pragma unroll
      for (int k = 0; k < NH; ++k) t[u][k] = __ldcg(&part[(b + u * kBlock) * NH + k]);
      r = u + 1;
    }
#pragma unroll
  for (int u = 0; u < 3; ++u)
    if (u < r) {
#pragma unroll
      for (int k = 0; k < NH; ++k) s[k] += t[u][k];
    }
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

#ifndef DOPT_TAIL_PROBE  // diagnostics build: timestamps of the reduction tail in the workspace
#define DOPT_TAIL_PROBE 0   // (tools/tail_probe.py; profiles/r02ad_*)
#endif
__device__ __forceinline__ unsigned long long probe_gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
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
  // Dynamic tail (large trees, hyper-gradient mode): the last kDynTailPct
  // percent of the vectors are split into chunks that blocks claim with an
  // atomic counter once their static share is done, so blocks on slower SMs
  // do not stretch the kernel's end. Each chunk's partial sum has its own
  // slot and is computed identically whichever block takes it: the total
  // stays a fixed-order, bitwise-reproducible sum. (Measured on B200: +1-2%
  // at 2^28 elements, -0.5% at the 11.7M-element C2 tree, hence the floor.)
  int64_t nstatic = nvec, nchunks = 0, chunk = kBlock;
  if (Op::NH > 0 && want_hp && nvec >= kDynTailMinVec) {
    const int64_t dyn = nvec * kDynTailPct / 100;
    const int64_t room = kMaxParts - gridDim.x;
    chunk = ((dyn / 256 + kBlock - 1) / kBlock) * kBlock;
    if (chunk < kBlock) chunk = kBlock;
    nchunks = room > 0 ? dyn / chunk : 0;
    if (nchunks > room) nchunks = room;
    nstatic = nvec - nchunks * chunk;
  }
  pdl_wait();
#if DOPT_TAIL_PROBE
  if (threadIdx.x == 0 && a.partials) a.partials[8192 + blockIdx.x] = (double)probe_gt();
#endif
#if DOPT_SPAN
  process_spans<Op, ST, U>(op, a, nstatic, tid, nthreads, acc, want_hp);
#else
  process_vectors<Op, ST, U>(op, a, 0, nstatic, tid, nthreads, acc, want_hp);
#endif
  if (nchunks == 0) pdl_trigger();
#if DOPT_TAIL_PROBE
  __syncthreads();
  if (threadIdx.x == 0 && a.partials) a.partials[12288 + blockIdx.x] = (double)probe_gt();
  long long c0 = clock64();
#endif
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
    if (nchunks > 0) {  // claim dynamic chunks until none is left
      __shared__ int64_t s_c;
      for (;;) {
        if (threadIdx.x == 0) s_c = (int64_t)atomicAdd(a.counter + 1, 1u);
        __syncthreads();
        const int64_t c = s_c;
        __syncthreads();
        if (c >= nchunks) break;
        double a2[NH];
#pragma unroll
        for (int k = 0; k < NH; ++k) a2[k] = 0.0;
        const int64_t v0 = nstatic + c * chunk;
        process_vectors<Op, ST, U>(op, a, v0, v0 + chunk, threadIdx.x, kBlock, a2, want_hp);
        block_sum<NH>(a2, sm);
        if (threadIdx.x == 0) {
#pragma unroll
          for (int k = 0; k < NH; ++k) a.partials[((int64_t)gridDim.x + c) * NH + k] = a2[k];
        }
      }
      pdl_trigger();
    }
#if DOPT_TAIL_PROBE
    long long c1 = clock64();
#endif
    const bool is_last = last_block(a.counter, gridDim.x);
#if DOPT_TAIL_PROBE
    long long c2 = clock64();
#endif
    if (is_last) {
      double s[NH];
#pragma unroll
      for (int k = 0; k < NH; ++k) s[k] = 0.0;
      const int64_t nparts = (int64_t)gridDim.x + nchunks;  // blocks, then chunks
      sum_partials<NH>(a.partials, nparts, s);
#if DOPT_TAIL_PROBE
      long long c3 = clock64();
#endif
      block_sum<NH>(s, sm);
      if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < NH; ++k)
          if (a.d_hp) a.d_hp[k] = s[k];
        a.counter[0] = 0u;
        a.counter[1] = 0u;
#if DOPT_TAIL_PROBE  // uniform-mode workspace slots beyond 4 x 4096 are free
        const long long c4 = clock64();
        a.partials[16384 + 0] = (double)(c1 - c0);  // block sum + partial store
        a.partials[16384 + 1] = (double)(c2 - c1);  // arrival ticket
        a.partials[16384 + 2] = (double)(c3 - c2);  // partial loads
        a.partials[16384 + 3] = (double)(c4 - c3);  // final block sum + store
        a.partials[16384 + 4] = (double)probe_gt();
        a.partials[16384 + 5] = (double)blockIdx.x;
#endif
      }
    }
  }
}

// --------------------------------------------- cp.async pipelined kernel
// The uniform kernel with the loads of vector v + nthreads in flight (as
// cp.async copies into this thread's shared-memory slots) while vector v is
// computed: the bytes in flight per warp no longer drop to zero during the
// math, without holding a second vector in registers. Dynamic smem:
// [2 stages][NIN][kBlock] 16-byte slots.
template <class Op, class ST>
__device__ __forceinline__ void pipe_issue(const StepArgs<Op::NIN, Op::NOUT>& a, int64_t v,
                                           float4* slot /* stage base + threadIdx.x */) {
#pragma unroll
  for (int i = 0; i < Op::NIN; ++i) {
    if (a.in[i]) {
      if (Op::in_state(i) && sizeof(ST) == 2)
        cp_async8(slot + i * kBlock, static_cast<const uint2*>(a.in[i]) + v);
      else
        cp_async16(slot + i * kBlock, static_cast<const float4*>(a.in[i]) + v);
    }
  }
}

template <class Op, class ST>
__device__ __forceinline__ void pipe_read(const StepArgs<Op::NIN, Op::NOUT>& a,
                                          const float4* slot, float (&x)[Op::NIN][4]) {
#pragma unroll
  for (int i = 0; i < Op::NIN; ++i) {
    if (a.in[i]) {
      if (Op::in_state(i) && sizeof(ST) == 2) {
        const uint2 t = *reinterpret_cast<const uint2*>(slot + i * kBlock);
        x[i][0] = __uint_as_float(t.x << 16);
        x[i][1] = __uint_as_float(t.x & 0xFFFF0000u);
        x[i][2] = __uint_as_float(t.y << 16);
        x[i][3] = __uint_as_float(t.y & 0xFFFF0000u);
      } else {
        const float4 t = slot[i * kBlock];
        x[i][0] = t.x; x[i][1] = t.y; x[i][2] = t.z; x[i][3] = t.w;
      }
    } else {
      x[i][0] = x[i][1] = x[i][2] = x[i][3] = 0.f;
    }
  }
}

template <class Op, class ST, int MINB>
__global__ void __launch_bounds__(kBlock, MINB) step_pipe(const Op op,
                                                    const StepArgs<Op::NIN, Op::NOUT> a) {
  constexpr int NH = Op::NH > 0 ? Op::NH : 1;
  const bool want_hp = Op::NH > 0 && a.want_hp;
  extern __shared__ float4 s_pipe[];
  float4* slot0 = s_pipe + threadIdx.x;
  float4* slot1 = s_pipe + Op::NIN * kBlock + threadIdx.x;
  double acc[NH];
#pragma unroll
  for (int k = 0; k < NH; ++k) acc[k] = 0.0;

  const int64_t nvec = a.numel >> 2;
  const int64_t nthreads = (int64_t)gridDim.x * kBlock;
  int64_t v = (int64_t)blockIdx.x * kBlock + threadIdx.x;
  pdl_wait();
  if (v < nvec) pipe_issue<Op, ST>(a, v, slot0);
  cp_async_commit();
  bool odd = false;
  for (; v < nvec; v += nthreads) {
    const int64_t vn = v + nthreads;
    if (vn < nvec) pipe_issue<Op, ST>(a, vn, odd ? slot0 : slot1);
    cp_async_commit();
    cp_async_wait<1>();  // this thread's copies of vector v have landed
    float x[Op::NIN][4];
    pipe_read<Op, ST>(a, odd ? slot1 : slot0, x);
    compute_store_vec<Op, ST>(op, a, v, x, acc, want_hp);
    odd = !odd;
  }
  cp_async_wait<0>();
  pdl_trigger();
  const int64_t tail0 = nvec << 2;
  if (blockIdx.x == gridDim.x - 1 && tail0 + threadIdx.x < a.numel)
    process_elem<Op, ST>(op, a, tail0 + threadIdx.x, acc, want_hp);

  if constexpr (Op::NH > 0) {
    if (!want_hp) return;
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
      sum_partials<NH>(a.partials, gridDim.x, s);
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

// ---------------------------------------------------------- leaf mode
// Pieces. The flat element range is cut into chunks of kChunk elements and
// every chunk into its intersections with the leaves. Piece (chunk c, leaf
// l) owns partial slot c + l: leaves are contiguous and ordered, so two
// non-empty pieces never share a slot, and leaf l's pieces are the
// consecutive slots [c_first(l) + l, c_last(l) + l] -- no scan and no table.
// The same rule one level up (super-chunks of 32 chunks) gives the slots of
// the second level. So the streaming kernel keeps the uniform kernel's
// grid-stride over equal work items (chunks; leaf count is free), and the
// per-leaf sums are two short fixed-order folds (leaf_fold, leaf_finalize).
__device__ __forceinline__ int64_t leaf_of(const int64_t* off, int64_t nl, int64_t e) {
  // the non-empty leaf holding element e: last l with off[l] <= e
  int64_t lo = 0, hi = nl - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (off[mid] <= e) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Elements [s, e) (one piece, <= kChunk) by the 32 lanes of a warp.
template <class Op, class ST, int U>
__device__ __forceinline__ void process_piece(const Op& op, const StepArgs<Op::NIN, Op::NOUT>& a,
                                              int64_t s, int64_t e, int lane, double* acc,
                                              bool want_hp) {
  const int64_t va = (s + 3) >> 2, vb = e >> 2;
  if (va < vb) {
    process_vectors<Op, ST, U>(op, a, va, vb, lane, 32, acc, want_hp);
    if (s + lane < (va << 2)) process_elem<Op, ST>(op, a, s + lane, acc, want_hp);
    if ((vb << 2) + lane < e) process_elem<Op, ST>(op, a, (vb << 2) + lane, acc, want_hp);
  } else {
    for (int64_t i = s + lane; i < e; i += 32) process_elem<Op, ST>(op, a, i, acc, want_hp);
  }
}

// Dynamic smem: the offset table (n_leaves + 1) when n_leaves <= kMaxLeafSmem,
// else the binary searches read it from global memory (L1-cached).
template <class Op, class ST, int U, int MINB>
__global__ void __launch_bounds__(kBlock, MINB) step_leaf(const Op op,
                                                    const StepArgs<Op::NIN, Op::NOUT> a) {
  constexpr int NH = Op::NH > 0 ? Op::NH : 1;
  const bool want_hp = Op::NH > 0 && a.want_hp;
  extern __shared__ int64_t s_dyn[];
  const int64_t nl = a.n_leaves;
  const bool staged = nl <= kMaxLeafSmem;
  pdl_wait();
  if (staged) {
    for (int64_t l = threadIdx.x; l <= nl; l += kBlock) s_dyn[l] = __ldg(&a.offsets[l]);
    __syncthreads();
  }
  const int64_t* off = staged ? s_dyn : a.offsets;
  const int lane = threadIdx.x & 31;
  const int64_t nchunks = n_chunks_of(a.numel), nwarps = (int64_t)gridDim.x * kWarps;
  for (int64_t c = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); c < nchunks; c += nwarps) {
    const int64_t c1 = min((c + 1) << kChunkShift, a.numel);
    int64_t s = c << kChunkShift;
    int64_t l = leaf_of(off, nl, s);
    while (true) {
      const int64_t e = min(c1, off[l + 1]);
      Op opt = op;  // the piece's leaf learning rate (per-leaf lr variants)
      if (a.lr_leaf) opt.set_lr((typename Op::CT)a.lr_leaf[l]);
      double acc[NH];
#pragma unroll
      for (int k = 0; k < NH; ++k) acc[k] = 0.0;
      process_piece<Op, ST, U>(opt, a, s, e, lane, acc, want_hp);
      if (want_hp) {
#pragma unroll
        for (int k = 0; k < NH; ++k) acc[k] = warp_sum(acc[k]);
        if (lane == 0)
#pragma unroll
          for (int k = 0; k < NH; ++k) a.partials[(c + l) * NH + k] = acc[k];
      }
      if (e >= c1) break;
      s = e;
      do { ++l; } while (off[l + 1] <= s);  // next non-empty leaf
    }
  }
  pdl_trigger();
}

// Level 2: one warp per super-chunk sc; for every leaf l meeting it, lane j
// takes chunk 32 sc + j's slot (c + l) and the xor-shuffle sum goes to slot
// sc + l of part2.
template <int NH>
__global__ void __launch_bounds__(kBlock) leaf_fold(const double* part1, const int64_t* off,
                                                    int64_t nl, int64_t numel, double* part2) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t sc = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (sc < n_supers_of(numel)) {
    const int64_t e1 = min((sc + 1) << kSuperShift, numel);
    const int64_t c = (sc << (kSuperShift - kChunkShift)) + lane;
    const bool chunk_ok = (c << kChunkShift) < e1;
    int64_t s = sc << kSuperShift;
    int64_t l = leaf_of(off, nl, s);
    while (true) {
      const int64_t lb = __ldg(&off[l]), le = __ldg(&off[l + 1]);
      const bool in = chunk_ok && c >= (lb >> kChunkShift) && c <= ((le - 1) >> kChunkShift);
      double v[NH];
#pragma unroll
      for (int k = 0; k < NH; ++k) v[k] = in ? __ldcg(&part1[(c + l) * NH + k]) : 0.0;
#pragma unroll
      for (int k = 0; k < NH; ++k) v[k] = warp_sum(v[k]);
      if (lane == 0)
#pragma unroll
        for (int k = 0; k < NH; ++k) part2[(sc + l) * NH + k] = v[k];
      if (le >= e1) break;
      s = le;
      do { ++l; } while (__ldg(&off[l + 1]) <= s);
    }
  }
  pdl_trigger();
}

// Level 3: one warp per leaf sums its super-chunk slots (lanes stride, then
// xor-shuffle) into d_hp_leaf; one fp64 partial per block of those sums (in
// leaf order) and the last block sums the partials in block order into d_hp.
// Every sum has a fixed order: bitwise reproducible.
template <int NH>
__global__ void __launch_bounds__(kBlock) leaf_finalize(const double* part2, const int64_t* off,
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
    const int64_t lb = __ldg(&off[l]), le = __ldg(&off[l + 1]);
    if (le > lb) {
      const int64_t sb = (le - 1) >> kSuperShift;
#pragma unroll 4
      for (int64_t sc = (lb >> kSuperShift) + lane; sc <= sb; sc += 32)
#pragma unroll
        for (int k = 0; k < NH; ++k) s[k] += __ldcg(&part2[(sc + l) * NH + k]);
    }
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
