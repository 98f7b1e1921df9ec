// tc_gemm.cuh -- fp32-accurate batched GEMM on the 5th-generation tensor
// cores (tcgen05, kind::tf32) by 3xTF32 splitting, for the MAML network's
// convolution contractions (include/mamlnet.h, net_tc_gemm).
//
//   D[t](m, n) = sum_k A[t](m, k) * B[t](n, k)   (+ bias[t][n])
//
// Each fp32 operand element x is split while it is staged into shared
// memory: hi = rna_tf32(x), lo = rna_tf32(x - hi) (x - hi is exact in fp32),
// and the tile product is accumulated in TMEM (fp32) as
// hi*hi + hi*lo + lo*hi: the dropped lo*lo term and the rounding of lo are
// ~2^-21 relative, i.e. fp32-GEMM accuracy, which the second-order MAML
// meta-gradient needs (single-pass TF32 is ~2^-11). Operands are read with
// coalesced global loads along whichever axis is contiguous in memory and
// stored into the 128B-swizzled K-major UMMA canonical layout either way (a
// thread holding 4 consecutive k of one row stores one 16-byte vector; the
// swizzle makes both store patterns bank-conflict-free), so no transposing
// pass is needed for any of the three convolution products.
//
// CTA: 128 threads, tile 128 (m, = UMMA M and the TMEM lanes) x 64 (n, UMMA
// N, 64 TMEM columns) x 32 (k per stage), two shared-memory stages: the
// threads split and store stage s+1 while the single elected thread's 12
// tcgen05.mma (4 k-steps x 3 products) of stage s run; tcgen05.commit on a
// per-stage mbarrier releases a stage and its TMEM accumulator (two 64-column
// accumulators, one per stage, each started fresh per 32-k block). While the
// MMAs of block i run, every thread folds block i-1's accumulator into 64
// fp32 registers with tcgen05.ld 32x32b (warp w owns lanes 32w..32w+31):
// the tensor core's truncating accumulation is confined to 96 products and
// the long sum is IEEE fp32 (measured: 3xTF32 error grows linearly with K
// when the whole K is accumulated in TMEM). Epilogue: optional bias,
// coalesced stores along m.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace tcg {

constexpr int BM = 128, BN = 64, BK = 32, THREADS = 128;
constexpr int A_BYTES = BM * BK * 4;  // 16 KB per split half
constexpr int B_BYTES = BN * BK * 4;  // 8 KB
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
constexpr int SMEM_BYTES = 2 * STAGE_BYTES + 1024 + 64;  // + 1024-B alignment slack + barriers

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// byte offset of (row r, k) in a K-major SW128 tile: 8-row groups of 1024 B,
// each row 128 B = 32 k, 16-B chunks XOR-swizzled by the row within the group
__device__ __forceinline__ uint32_t off_k(int r, int k) {
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((((k >> 2) ^ (r & 7))) << 4) + (k & 3) * 4);
}
// UMMA shared-memory descriptor (SM100: version 1), 128B swizzle
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

template <bool A_MN, bool B_MN>
__device__ __forceinline__ constexpr uint32_t idesc() {
  return (1u << 4)                     // D fp32
         | (2u << 7) | (2u << 10)      // A, B tf32
         | ((A_MN ? 1u : 0u) << 15) | ((B_MN ? 1u : 0u) << 16)
         | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity));
}

struct Args {
  int M, N, K;           // per batch
  const float* A;        // A(m, k) at A + m*sAm + k*sAk (+ t*bA)
  int64_t sAm, sAk, bA;
  const float* B;        // B(n, k) at B + n*sBn + k*sBk (+ t*bB)
  int64_t sBn, sBk, bB;
  float* D;              // D(m, n) at D + m + n*ldD (+ t*bD) (+ s*sS when split)
  int64_t ldD, bD, sS;
  const float* bias;     // bias[t*N + n] or nullptr
  int kchunk;            // k per split (multiple of BK)
  int mtiles;
};

template <bool A_MN, bool B_MN>
__global__ void __launch_bounds__(THREADS, 1) tc3_gemm_kernel(const Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(smem + 2 * STAGE_BYTES);  // [0], [1]: stage free
  uint32_t* tslot = (uint32_t*)(bars + 2);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t = blockIdx.z, s = blockIdx.y;
  const int mt = blockIdx.x % a.mtiles, nt = blockIdx.x / a.mtiles;
  const int m0 = mt * BM, n0 = nt * BN;
  const int kbeg = s * a.kchunk, kend = min(a.K, kbeg + a.kchunk);
  const float* A = a.A + (int64_t)t * a.bA;
  const float* B = a.B + (int64_t)t * a.bB;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
        smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tslot;

  const int nkb = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
  float racc[BN];
#pragma unroll
  for (int j = 0; j < BN; ++j) racc[j] = 0.f;
  auto fold = [&](int blk) {  // wait for block blk's MMAs, add its accumulator
    mbar_wait(&bars[blk & 1], (blk >> 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
    for (int c = 0; c < BN; c += 16) {
      uint32_t v[16];
      const uint32_t taddr =
          tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)((blk & 1) * BN + c);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
          "%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
            "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
      for (int j = 0; j < 16; ++j) racc[c + j] += __uint_as_float(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
  };
  for (int it = 0; it < nkb; ++it) {
    const int st = it & 1;
    if (it >= 2) mbar_wait(&bars[st], ((it - 2) >> 1) & 1);
    uint8_t* base = smem + st * STAGE_BYTES;
    uint8_t *ahi = base, *alo = base + A_BYTES, *bhi = base + 2 * A_BYTES,
            *blo = base + 2 * A_BYTES + B_BYTES;
    const int k0 = kbeg + it * BK;
    // ---- A tile: 128 x 32, stored K-major (SW128) in both orientations
    if (A_MN) {
      // thread = row m, 32 k's: each load instruction is coalesced along m;
      // then eight 16-byte stores per half (conflict-free through the swizzle)
      const int m = m0 + tid;
      const bool mok = m < a.M;
#pragma unroll
      for (int c = 0; c < BK / 4; ++c) {
        float x[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int k = k0 + 4 * c + j;
          x[j] = (mok && k < kend) ? __ldg(A + (int64_t)m * a.sAm + (int64_t)k * a.sAk) : 0.f;
        }
        uint4 h, l;
        h.x = to_tf32(x[0]), l.x = to_tf32(x[0] - __uint_as_float(h.x));
        h.y = to_tf32(x[1]), l.y = to_tf32(x[1] - __uint_as_float(h.y));
        h.z = to_tf32(x[2]), l.z = to_tf32(x[2] - __uint_as_float(h.z));
        h.w = to_tf32(x[3]), l.w = to_tf32(x[3] - __uint_as_float(h.w));
        const uint32_t o = off_k(tid, 4 * c);
        *(uint4*)(ahi + o) = h;
        *(uint4*)(alo + o) = l;
      }
    } else {
      const int k = k0 + lane;
      const bool kok = k < kend;
#pragma unroll 8
      for (int i = 0; i < BM / 4; ++i) {
        const int r = warp + 4 * i, m = m0 + r;
        const float x = (kok && m < a.M) ? __ldg(A + (int64_t)m * a.sAm + (int64_t)k * a.sAk) : 0.f;
        const uint32_t h = to_tf32(x), l = to_tf32(x - __uint_as_float(h));
        const uint32_t o = off_k(r, lane);
        *(uint32_t*)(ahi + o) = h;
        *(uint32_t*)(alo + o) = l;
      }
    }
    // ---- B tile: 64 x 32, K-major
    if (B_MN) {
      const int r = tid & 63, n = n0 + r, kh = (tid >> 6) * 16;
      const bool nok = n < a.N;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float x[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int k = k0 + kh + 4 * c + j;
          x[j] = (nok && k < kend) ? __ldg(B + (int64_t)n * a.sBn + (int64_t)k * a.sBk) : 0.f;
        }
        uint4 h, l;
        h.x = to_tf32(x[0]), l.x = to_tf32(x[0] - __uint_as_float(h.x));
        h.y = to_tf32(x[1]), l.y = to_tf32(x[1] - __uint_as_float(h.y));
        h.z = to_tf32(x[2]), l.z = to_tf32(x[2] - __uint_as_float(h.z));
        h.w = to_tf32(x[3]), l.w = to_tf32(x[3] - __uint_as_float(h.w));
        const uint32_t o = off_k(r, kh + 4 * c);
        *(uint4*)(bhi + o) = h;
        *(uint4*)(blo + o) = l;
      }
    } else {
      const int k = k0 + lane;
      const bool kok = k < kend;
#pragma unroll 8
      for (int i = 0; i < BN / 4; ++i) {
        const int r = warp + 4 * i, n = n0 + r;
        const float x = (kok && n < a.N) ? __ldg(B + (int64_t)n * a.sBn + (int64_t)k * a.sBk) : 0.f;
        const uint32_t h = to_tf32(x), l = to_tf32(x - __uint_as_float(h));
        const uint32_t o = off_k(r, lane);
        *(uint32_t*)(bhi + o) = h;
        *(uint32_t*)(blo + o) = l;
      }
    }
    asm volatile("fence.proxy.async.shared::cta;");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t ah = smem_u32(ahi), al = smem_u32(alo), bh = smem_u32(bhi), bl = smem_u32(blo);
      const uint32_t tacc = tmem + (uint32_t)(st * BN);  // accumulator of this stage
      constexpr uint32_t id = idesc<false, false>();  // both operands K-major in smem
#pragma unroll
      for (int kk = 0; kk < BK / 8; ++kk) {
        // k-step of 8 tf32 = 32 B inside the 128-B swizzle atom
        const uint64_t dah = sdesc(ah + kk * 32, 16, 1024), dal = sdesc(al + kk * 32, 16, 1024);
        const uint64_t dbh = sdesc(bh + kk * 32, 16, 1024), dbl = sdesc(bl + kk * 32, 16, 1024);
        const uint32_t acc0 = kk > 0 ? 1u : 0u;  // a fresh accumulator per 32-k block
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tacc),
            "l"(dah), "l"(dbh), "r"(id), "r"(acc0));
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tacc),
            "l"(dah), "l"(dbl), "r"(id), "r"(1u));
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tacc),
            "l"(dal), "l"(dbh), "r"(id), "r"(1u));
      }
      asm volatile(
          "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
              smem_u32(&bars[st])));
    }
    // while the MMAs of this block run: fold the previous block's accumulator
    // into fp32 registers (round-to-nearest adds: the tensor core's own
    // accumulation error stays confined to 32-k blocks)
    if (it >= 1) fold(it - 1);
  }
  if (nkb >= 1) fold(nkb - 1);

  // ---- epilogue: thread = row m (TMEM lane 32w + lane), 64 columns
  const int m = m0 + warp * 32 + lane;
  float* D = a.D + (int64_t)t * a.bD + (int64_t)s * a.sS;
  const float* bias = a.bias ? a.bias + (int64_t)t * a.N : nullptr;
  if (m < a.M) {
#pragma unroll
    for (int j = 0; j < BN; ++j) {
      const int n = n0 + j;
      if (n < a.N) D[(int64_t)m + (int64_t)n * a.ldD] = bias ? racc[j] + bias[n] : racc[j];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

}  // namespace tcg
