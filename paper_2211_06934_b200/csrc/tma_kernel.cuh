// tma_kernel.cuh -- TMA-bulk pipelined variant of the one-pass step kernel.
//
// Blackwell-native streaming: one persistent CTA per SM
// = 8 consumer warps + 1 producer warp. The producer's elected lane streams
// every input array of a kTmaTile-element tile into a STAGES-deep shared
// memory ring with 1-D bulk copies (cp.async.bulk ... mbarrier::complete_tx,
// SASS UBLKCP), so up to STAGES tiles of all inputs are in flight per SM
// without holding registers; consumers wait on the tile's full barrier,
// compute from shared memory, store results straight to HBM (16-byte
// streaming stores) and release the slot on its empty barrier. The hyper-
// gradient reduction is the same fixed-order block partial + last-block sum
// as step_uniform, so results are identical in structure.
#pragma once
#include <stdint.h>

#include "step_kernel.cuh"

namespace dopt {

// Consumer threads per CTA (NCONS) and tile = 4 * NCONS elements are
// template parameters; the producer is one extra warp.

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <class Op, class ST, int NCONS>
struct TmaLayout {
  static constexpr int kTile = 4 * NCONS;
  // bytes of one tile of input array i in shared memory
  static __host__ __device__ constexpr uint32_t in_bytes(int i) {
    return (uint32_t)kTile * (Op::in_state(i) ? (uint32_t)sizeof(ST) : 4u);
  }
  static __host__ __device__ constexpr uint32_t stage_bytes() {
    uint32_t b = 0;
    for (int i = 0; i < Op::NIN; ++i) b += in_bytes(i);
    return b;
  }
};

template <class Op, class ST, int STAGES, int NCONS>
__host__ __device__ constexpr size_t tma_smem_bytes() {
  return (size_t)STAGES * TmaLayout<Op, ST, NCONS>::stage_bytes() + 2 * STAGES * sizeof(uint64_t) + 128;
}

// smem vector of 4 elements (fp32 16 B, bf16 8 B) -> float[4]
__device__ __forceinline__ void lds4(const float* p, float (&o)[4]) {
  float4 t = *reinterpret_cast<const float4*>(p);
  o[0] = t.x; o[1] = t.y; o[2] = t.z; o[3] = t.w;
}
__device__ __forceinline__ void lds4(const bf16* p, float (&o)[4]) {
  uint2 t = *reinterpret_cast<const uint2*>(p);
  o[0] = __uint_as_float(t.x << 16);
  o[1] = __uint_as_float(t.x & 0xFFFF0000u);
  o[2] = __uint_as_float(t.y << 16);
  o[3] = __uint_as_float(t.y & 0xFFFF0000u);
}

template <class Op, class ST, int STAGES, int NCONS, int MINB>
__global__ void __launch_bounds__(NCONS + 32, MINB)
    step_tma(const Op op, const StepArgs<Op::NIN, Op::NOUT> a) {
  typedef TmaLayout<Op, ST, NCONS> Lay;
  constexpr int kTmaConsumers = NCONS;
  constexpr int kTmaThreads = NCONS + 32;
  constexpr int kTmaTile = Lay::kTile;
  constexpr int NH = Op::NH > 0 ? Op::NH : 1;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)STAGES * Lay::stage_bytes());
  uint64_t* empty = full + STAGES;

  const bool want_hp = Op::NH > 0 && a.want_hp;
  const int64_t numel = a.numel;
  const int64_t n_tiles = (numel + kTmaTile - 1) / kTmaTile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  pdl_wait();
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTmaConsumers / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  double acc[NH];
#pragma unroll
  for (int k = 0; k < NH; ++k) acc[k] = 0.0;

  if (warp == kTmaConsumers / 32) {
    // ------------------------------------------------------- producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int64_t e0 = tile * kTmaTile;
        int64_t cnt = numel - e0 < kTmaTile ? numel - e0 : kTmaTile;
        cnt &= ~int64_t(7);  // bulk copies in 16-byte units (8 bf16 / 4 fp32)
        mbar_wait(&empty[stage], phase ^ 1);
        uint32_t bytes = 0;
#pragma unroll
        for (int i = 0; i < Op::NIN; ++i)
          if (a.in[i]) bytes += (uint32_t)cnt * (Op::in_state(i) ? (uint32_t)sizeof(ST) : 4u);
        mbar_expect_tx(&full[stage], bytes);
        if (cnt > 0) {
          unsigned char* base = smem + (size_t)stage * Lay::stage_bytes();
#pragma unroll
          for (int i = 0; i < Op::NIN; ++i) {
            if (a.in[i]) {
              const uint32_t eb = Op::in_state(i) ? (uint32_t)sizeof(ST) : 4u;
              const unsigned char* src = static_cast<const unsigned char*>(a.in[i]) + e0 * eb;
              bulk_g2s(base, src, (uint32_t)cnt * eb, &full[stage]);
            }
            base += Lay::in_bytes(i);
          }
        }
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else {
    // ------------------------------------------------------ consumers
    typedef typename Op::CT CT;
    int stage = 0;
    uint32_t phase = 0;
    const int t = threadIdx.x;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      const int64_t e0 = tile * kTmaTile;
      const int64_t rem = numel - e0;
      const int64_t cnt = (rem < kTmaTile ? rem : kTmaTile) & ~int64_t(7);
      mbar_wait(&full[stage], phase);
      const int64_t el = 4 * t;  // this thread's 4 elements within the tile
      const bool whole = el + 4 <= cnt;
      float x[Op::NIN][4];
      if (whole) {
        const unsigned char* base = smem + (size_t)stage * Lay::stage_bytes();
#pragma unroll
        for (int i = 0; i < Op::NIN; ++i) {
          if (a.in[i]) {
            if (Op::in_state(i))
              lds4(reinterpret_cast<const ST*>(base) + el, x[i]);
            else
              lds4(reinterpret_cast<const float*>(base) + el, x[i]);
          } else {
            x[i][0] = x[i][1] = x[i][2] = x[i][3] = 0.f;
          }
          base += Lay::in_bytes(i);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);  // slot free: data is in registers
      if (whole) {
        compute_store_vec<Op, ST>(op, a, (e0 >> 2) + t, x, acc, want_hp);
      } else {
        // ragged end of the last tile (< 8 elements past the bulk copy)
        for (int k = 0; k < 4; ++k) {
          const int64_t i = e0 + el + k;
          if (el + k >= cnt && i < numel) process_elem<Op, ST>(op, a, i, acc, want_hp);
        }
      }
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }
  }

  if constexpr (Op::NH > 0) {
    if (!want_hp) return;
    __shared__ double sm[NH][kTmaThreads / 32];
    // block sum over 9 warps (producer contributes 0), fixed order
    {
#pragma unroll
      for (int k = 0; k < NH; ++k) {
        double s = warp_sum(acc[k]);
        if (lane == 0) sm[k][warp] = s;
      }
      __syncthreads();
      if (warp == 0) {
#pragma unroll
        for (int k = 0; k < NH; ++k) {
          double s = lane < kTmaThreads / 32 ? sm[k][lane] : 0.0;
          acc[k] = warp_sum(s);
        }
      }
      __syncthreads();
    }
    if (threadIdx.x == 0)
#pragma unroll
      for (int k = 0; k < NH; ++k) a.partials[(int64_t)blockIdx.x * NH + k] = acc[k];
    if (last_block(a.counter, gridDim.x)) {
      double s[NH];
#pragma unroll
      for (int k = 0; k < NH; ++k) s[k] = 0.0;
      for (int64_t b = threadIdx.x; b < gridDim.x; b += kTmaThreads)
#pragma unroll
        for (int k = 0; k < NH; ++k) s[k] += __ldcg(&a.partials[b * NH + k]);
#pragma unroll
      for (int k = 0; k < NH; ++k) {
        double w = warp_sum(s[k]);
        if (lane == 0) sm[k][warp] = w;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < NH; ++k) {
          double tot = 0.0;
          for (int w = 0; w < kTmaThreads / 32; ++w) tot += sm[k][w];
          if (a.d_hp) a.d_hp[k] = tot;
        }
        *a.counter = 0u;
      }
    }
  }
}

}  // namespace dopt
