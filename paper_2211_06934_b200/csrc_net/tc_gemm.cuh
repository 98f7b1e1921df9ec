// tc_gemm.cuh -- fp32-accurate batched GEMM on the 5th-generation tensor
// cores (tcgen05, kind::tf32) by 3xTF32 splitting, for the MAML network's
// convolution contractions (include/mamlnet.h, net_tc_gemm).
//
//   D[t](m, n) = sum_k A[t](m, k) * B[t](n, k)   (+ bias[t][n])
//
// Each fp32 operand element x is split while it is staged into shared
// memory: hi = x truncated to tf32, lo = x - hi (exact in fp32), and the
// tile product is accumulated in TMEM (fp32) as hi*hi + hi*lo + lo*hi: the
// dropped lo*lo term and the tensor core's truncation of lo are ~2^-20
// relative, i.e. fp32-GEMM accuracy, which the second-order MAML
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

constexpr int BM = 128, BN = 64, BK = 32, RSTAGES = 4;
// warp roles: 0-3 copy + split (LOADERS threads), 4-7 fold + epilogue (TMEM
// lane quarter = warp % 4), 8 MMA issue
constexpr int LOADERS = 128, THREADS = 288, EPI_WARP0 = 4, MMA_WARP = 8;
constexpr int A_BYTES = BM * BK * 4;  // 16 KB per split half
constexpr int B_BYTES = BN * BK * 4;  // 8 KB
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;

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
  int mtiles, splits, ntiles;
  int dbg;  // diagnostics only (NET_TC_DBG): 1 = no MMA, 2 = no split, 4 = no copies
};

// Raw fp32 tiles as copied (cp.async, zero-filled outside the matrix):
// m/n-contiguous operands as [k][R + 4], k-contiguous ones as [R][36]; the
// pads keep 16-byte alignment and make the split's 16-byte reads cover all
// banks per quarter-warp.
constexpr int RAW_A = (BK * (BM + 4) > BM * 36) ? BK * (BM + 4) : BM * 36;  // floats
constexpr int RAW_B = (BK * (BN + 4) > BN * 36) ? BK * (BN + 4) : BN * 36;
constexpr int RAW_STAGE = (RAW_A + RAW_B) * 4;
constexpr int FOLD = 4;  // k-blocks (4 x 32 k) accumulated in TMEM before an fp32 fold
// split stages + raw ring + 1024-B alignment slack + barriers / TMEM slot
constexpr int SMEM_BYTES = 2 * STAGE_BYTES + RSTAGES * RAW_STAGE + 1024 + 64;

__device__ __forceinline__ void cp_async(uint32_t dst, const float* src, int bytes, int cp) {
  if (cp == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(bytes));
}

// Per-thread copy plan for one operand tile of R rows x BK k: the thread's
// elements (or 4-wide chunks when V) are fixed across k-blocks, so offsets
// and row validity are computed once; per block only k changes.
template <bool MN, bool V, int R>
struct CopyPlan {
  static constexpr int RS = MN ? R + 4 : 36;                       // raw row stride
  static constexpr int UNITS = V ? R * BK / 4 : R * BK;            // chunks or elements
  static constexpr int PER = UNITS / LOADERS > 0 ? UNITS / LOADERS : 1;
  int64_t off[PER];   // global offset at k = 0 (floats)
  int kk[PER];        // k within the block
  int rows_left[PER]; // rows (MN) valid from this chunk's first row, <= 0 if none
  uint32_t dst[PER];  // smem byte offset within the raw tile
  bool live[PER];
  __device__ void init(int tid, int row0, int M, int64_t s_r, int64_t s_k) {
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int u = tid + LOADERS * j;
      live[j] = u < UNITS;
      int r, k;
      if (MN) {  // rows contiguous
        const int per_k = V ? R / 4 : R;
        r = (u % per_k) * (V ? 4 : 1), k = u / per_k;
        dst[j] = (uint32_t)(k * RS + r) * 4;
      } else {   // k contiguous
        const int per_r = V ? BK / 4 : BK;
        k = (u % per_r) * (V ? 4 : 1), r = u / per_r;
        dst[j] = (uint32_t)(r * RS + k) * 4;
      }
      kk[j] = k;
      rows_left[j] = M - (row0 + r);
      off[j] = (int64_t)(row0 + r) * s_r + (int64_t)k * s_k;
    }
  }
  __device__ __forceinline__ void issue(uint32_t base, const float* X, int k0, int kend,
                                        int64_t s_k) const {
    const int64_t kofs = (int64_t)k0 * s_k;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      if (!live[j]) continue;
      const int k = k0 + kk[j];
      int bytes;
      if (V) {
        if (MN) bytes = k < kend ? 4 * max(0, min(4, rows_left[j])) : 0;
        else bytes = rows_left[j] > 0 ? 4 * max(0, min(4, kend - k)) : 0;
      } else {
        bytes = (k < kend && rows_left[j] > 0) ? 4 : 0;
      }
      cp_async(base + dst[j], bytes ? X + off[j] + kofs : X, bytes, V ? 16 : 4);
    }
  }
};

// hi = x with the low 13 mantissa bits cleared (exactly representable in
// tf32), lo = x - hi (exact in fp32, |lo| < 2^-10 |x|); the tensor core reads
// lo's top 19 bits (truncation: <= 2^-20 |x|). Two instructions per element
// (cvt.rna.tf32 expands to a compare-and-branch sequence in SASS).
__device__ __forceinline__ uint32_t hi_bits(float x) { return __float_as_uint(x) & 0xFFFFE000u; }
__device__ __forceinline__ void split4(float4 x, uint4& h, uint4& l) {
  h.x = hi_bits(x.x), l.x = __float_as_uint(x.x - __uint_as_float(h.x));
  h.y = hi_bits(x.y), l.y = __float_as_uint(x.y - __uint_as_float(h.y));
  h.z = hi_bits(x.z), l.z = __float_as_uint(x.z - __uint_as_float(h.z));
  h.w = hi_bits(x.w), l.w = __float_as_uint(x.w - __uint_as_float(h.w));
}

// raw tile -> K-major SW128 hi / lo tiles (R rows x 32 k), by the LOADERS threads
template <bool MN, int R>
__device__ __forceinline__ void split_tile(const float* raw, uint8_t* hi, uint8_t* lo, int tid) {
  if (MN) {  // raw [k][R+4]: unit = (row quad q, k quad kq); 4x4 transpose in registers
    constexpr int RS = R + 4, NQ = R / 4;
#pragma unroll
    for (int u = tid; u < NQ * 8; u += LOADERS) {
      const int kq = u % 8, q = u / 8;
      float4 x[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) x[i] = *(const float4*)(raw + (4 * kq + i) * RS + 4 * q);
      const float4 cs[4] = {make_float4(x[0].x, x[1].x, x[2].x, x[3].x),
                            make_float4(x[0].y, x[1].y, x[2].y, x[3].y),
                            make_float4(x[0].z, x[1].z, x[2].z, x[3].z),
                            make_float4(x[0].w, x[1].w, x[2].w, x[3].w)};
#pragma unroll
      for (int jr = 0; jr < 4; ++jr) {
        uint4 h, l;
        split4(cs[jr], h, l);
        const uint32_t o = off_k(4 * q + jr, 4 * kq);
        *(uint4*)(hi + o) = h;
        *(uint4*)(lo + o) = l;
      }
    }
  } else {   // raw [R][36]: unit = (row, k quad), 16-byte reads along k
#pragma unroll
    for (int u = tid; u < R * 8; u += LOADERS) {
      const int r = u % R, kq = u / R;
      const float4 x = *(const float4*)(raw + r * 36 + 4 * kq);
      uint4 h, l;
      split4(x, h, l);
      const uint32_t o = off_k(r, 4 * kq);
      *(uint4*)(hi + o) = h;
      *(uint4*)(lo + o) = l;
    }
  }
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void loader_sync() {  // named barrier over the LOADERS threads
  asm volatile("bar.sync 1, %0;" ::"n"(LOADERS) : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar)));
}

struct Tile {  // one 128 x 64 output tile of one (batch, k-split)
  int t, s, m0, n0, kbeg, kend, nkb;
  __device__ Tile(const Args& a, int idx) {
    const int ntn = (a.N + BN - 1) / BN, S = a.splits;
    int r = idx;
    const int mt = r % a.mtiles;
    r /= a.mtiles;
    const int nt = r % ntn;
    r /= ntn;
    s = r % S;
    t = r / S;
    m0 = mt * BM, n0 = nt * BN;
    kbeg = s * a.kchunk, kend = min(a.K, kbeg + a.kchunk);
    nkb = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
  }
};

// Persistent and warp-specialised: CTA c walks tiles c, c + gridDim.x, ...
// as one stream of 32-k blocks. Copy/split warps (0-3) keep a 4-deep
// cp.async ring of raw fp32 tiles and write the split hi / lo stages; the MMA
// warp (8) issues 12 tcgen05.mma per block into one of two TMEM
// accumulators; fold/epilogue warps (4-7) add each finished group of FOLD
// blocks into fp32 registers and store finished tiles. The roles meet only
// at mbarriers (stage full / empty, accumulator full / empty), so copies,
// splitting, MMAs and epilogues of different blocks and tiles overlap.
template <bool A_MN, bool B_MN, bool VA, bool VB>
__global__ void __launch_bounds__(THREADS, 1) tc3_gemm_kernel(const Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* raw = smem + 2 * STAGE_BYTES;  // RSTAGES raw fp32 stages
  uint64_t* bars = (uint64_t*)(raw + RSTAGES * RAW_STAGE);
  uint64_t* hfull = bars;       // [2] split stage written (LOADERS arrivals)
  uint64_t* hempty = bars + 2;  // [2] split stage consumed (MMA commit)
  uint64_t* afull = bars + 4;   // [2] accumulator group done (MMA commit)
  uint64_t* aempty = bars + 6;  // [2] accumulator drained (4 epilogue warps)
  uint32_t* tslot = (uint32_t*)(bars + 8);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ntiles = a.ntiles;

  if (warp == EPI_WARP0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
        smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&hfull[0], LOADERS), mbar_init(&hfull[1], LOADERS);
    mbar_init(&hempty[0], 1), mbar_init(&hempty[1], 1);
    mbar_init(&afull[0], 1), mbar_init(&afull[1], 1);
    mbar_init(&aempty[0], 4), mbar_init(&aempty[1], 4);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tslot;

  if (warp < EPI_WARP0) {
    // ===================== copy + split warps =====================
    CopyPlan<A_MN, VA, BM> pa;
    CopyPlan<B_MN, VB, BN> pb;
    const uint32_t raw0 = smem_u32(raw);
    int itile = blockIdx.x, ikb = 0, iq = 0, ik0 = 0, ikend = 0, inkb = 0;
    const float *iA = nullptr, *iB = nullptr;
    auto iset = [&]() {
      while (itile < ntiles) {
        const Tile T(a, itile);
        if (T.nkb > 0) {
          pa.init(tid, T.m0, a.M, a.sAm, a.sAk);
          pb.init(tid, T.n0, a.N, a.sBn, a.sBk);
          iA = a.A + (int64_t)T.t * a.bA, iB = a.B + (int64_t)T.t * a.bB;
          ik0 = T.kbeg, ikend = T.kend, inkb = T.nkb;
          return;
        }
        itile += gridDim.x;
      }
    };
    iset();
    auto issue = [&]() {
      if (itile < ntiles) {
        const uint32_t ra = raw0 + (iq % RSTAGES) * RAW_STAGE;
        const int k0 = ik0 + ikb * BK;
        if (!(a.dbg & 4)) {
          pa.issue(ra, iA, k0, ikend, a.sAk);
          pb.issue(ra + RAW_A * 4, iB, k0, ikend, a.sBk);
        }
        ++iq;
        if (++ikb == inkb) {
          ikb = 0;
          itile += gridDim.x;
          iset();
        }
      }
      asm volatile("cp.async.commit_group;");  // one group per call (empty past the end)
    };
    for (int b = 0; b < RSTAGES - 1; ++b) issue();
    int q = 0;
    for (int ct = blockIdx.x; ct < ntiles; ct += gridDim.x) {
      const int nkb = Tile(a, ct).nkb;
      for (int kb = 0; kb < nkb; ++kb, ++q) {
        const int st = q & 1;
        issue();                                                    // block q + RSTAGES - 1
        asm volatile("cp.async.wait_group %0;" ::"n"(RSTAGES - 1));  // block q: own copies
        loader_sync();                                              // ... and everyone's
        if (q >= 2) mbar_wait(&hempty[st], ((q - 2) >> 1) & 1);     // MMAs of q-2 done
        const float* ra = (const float*)(raw + (q % RSTAGES) * RAW_STAGE);
        uint8_t* base = smem + st * STAGE_BYTES;
        if (!(a.dbg & 2)) {
          split_tile<A_MN, BM>(ra, base, base + A_BYTES, tid);
          split_tile<B_MN, BN>(ra + RAW_A, base + 2 * A_BYTES, base + 2 * A_BYTES + B_BYTES, tid);
        }
        asm volatile("fence.proxy.async.shared::cta;");
        mbar_arrive(&hfull[st]);
        loader_sync();  // raw stage q % RSTAGES fully read before it is refilled
      }
    }
    asm volatile("cp.async.wait_group 0;");
  } else if (warp == MMA_WARP) {
    // ===================== MMA issue (one thread) =====================
    if (lane == 0) {
      int q = 0, g = 0;
      constexpr uint32_t id = idesc<false, false>();  // both operands K-major in smem
      for (int ct = blockIdx.x; ct < ntiles; ct += gridDim.x) {
        const int nkb = Tile(a, ct).nkb;
        for (int kb = 0; kb < nkb; ++kb, ++q) {
          const int st = q & 1;
          const bool gstart = kb % FOLD == 0, gend = kb % FOLD == FOLD - 1 || kb == nkb - 1;
          mbar_wait(&hfull[st], (q >> 1) & 1);
          if (gstart && g >= 2) mbar_wait(&aempty[g & 1], ((g - 2) >> 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          uint8_t* base = smem + st * STAGE_BYTES;
          const uint32_t ah = smem_u32(base), al = ah + A_BYTES, bh = ah + 2 * A_BYTES,
                         bl = bh + B_BYTES;
          const uint32_t tacc = tmem + (uint32_t)((g & 1) * BN);
#pragma unroll
          for (int kk = 0; kk < ((a.dbg & 1) ? 0 : BK / 8); ++kk) {
            // k-step of 8 tf32 = 32 B inside the 128-B swizzle atom
            const uint64_t dah = sdesc(ah + kk * 32, 16, 1024), dal = sdesc(al + kk * 32, 16, 1024);
            const uint64_t dbh = sdesc(bh + kk * 32, 16, 1024), dbl = sdesc(bl + kk * 32, 16, 1024);
            const uint32_t acc0 = (!gstart || kk > 0) ? 1u : 0u;  // fresh per group
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
          umma_commit(&hempty[st]);
          if (gend) {
            umma_commit(&afull[g & 1]);
            ++g;
          }
        }
      }
    }
  } else if (warp >= EPI_WARP0 && warp < EPI_WARP0 + 4) {
    // ===================== fold + epilogue warps =====================
    const int lq = warp & 3;  // TMEM lane quarter this warp may access
    float racc[BN];
#pragma unroll
    for (int j = 0; j < BN; ++j) racc[j] = 0.f;
    int g = 0;
    for (int ct = blockIdx.x; ct < ntiles; ct += gridDim.x) {
      const Tile T(a, ct);
      const int ngroups = (T.nkb + FOLD - 1) / FOLD;
      for (int gi = 0; gi < ngroups; ++gi, ++g) {
        mbar_wait(&afull[g & 1], (g >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
        for (int c = 0; c < BN; c += 16) {
          uint32_t v[16];
          const uint32_t taddr = tmem + ((uint32_t)(lq * 32) << 16) + (uint32_t)((g & 1) * BN + c);
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,"
              "%12,%13,%14,%15}, [%16];"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
                "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
              : "r"(taddr));
          asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
          for (int j = 0; j < 16; ++j) racc[c + j] += __uint_as_float(v[j]);
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive(&aempty[g & 1]);
      }
      // tile done: store (or bias / zero for an empty k range)
      const int m = T.m0 + lq * 32 + lane;
      float* D = a.D + (int64_t)T.t * a.bD + (int64_t)T.s * a.sS;
      const float* bias = a.bias ? a.bias + (int64_t)T.t * a.N : nullptr;
      if (m < a.M) {
#pragma unroll
        for (int j = 0; j < BN; ++j) {
          const int n = T.n0 + j;
          if (n < a.N) D[(int64_t)m + (int64_t)n * a.ldD] = bias ? racc[j] + bias[n] : racc[j];
        }
      }
#pragma unroll
      for (int j = 0; j < BN; ++j) racc[j] = 0.f;
    }
    if (warp == EPI_WARP0) {  // every MMA has completed (last afull waited)
      asm volatile("tcgen05.fence::after_thread_sync;");
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
    }
  }
}

}  // namespace tcg
