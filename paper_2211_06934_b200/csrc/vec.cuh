// vec.cuh -- streaming 4-element vector access for fp32 and bf16 arrays.
//
// Every array of the step is read once and written once (no reuse), so all
// global traffic uses the streaming cache policy (.cs: evict-first) and
// 16-byte (fp32) / 8-byte (bf16) vector instructions; a warp moves 512 B
// (resp. 256 B) per instruction, fully coalesced. Loads are coherent (not
// .nc) because outputs may alias inputs exactly (diffopt.h conventions);
// each element is read before it is written, by the same thread.
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

namespace dopt {

typedef __nv_bfloat16 bf16;

// Cache-policy variants for tuning sweeps (tools/tune_build.py "ldN"/"stN"):
// loads 0 = .cs (default), 1 = plain, 3 = .lu; stores 0 = .cs (default),
// 1 = plain write-back, 3 = .cg.
#ifndef DOPT_LD_POLICY
#define DOPT_LD_POLICY 0
#endif
#ifndef DOPT_ST_POLICY
#define DOPT_ST_POLICY 0
#endif
template <class T>
__device__ __forceinline__ T ld_stream(const T* p) {
#if DOPT_LD_POLICY == 1
  return *p;
#elif DOPT_LD_POLICY == 3
  return __ldlu(p);
#else
  return __ldcs(p);
#endif
}
template <class T>
__device__ __forceinline__ void st_stream(T* p, T x) {
#if DOPT_ST_POLICY == 1
  *p = x;
#elif DOPT_ST_POLICY == 3
  __stcg(p, x);
#else
  __stcs(p, x);
#endif
}

// ---- 4 consecutive elements at vector index v (element 4v .. 4v+3)
__device__ __forceinline__ void load4(const float* p, int64_t v, float (&o)[4]) {
  float4 t = ld_stream(reinterpret_cast<const float4*>(p) + v);
  o[0] = t.x; o[1] = t.y; o[2] = t.z; o[3] = t.w;
}

__device__ __forceinline__ void load4(const bf16* p, int64_t v, float (&o)[4]) {
  uint2 t = ld_stream(reinterpret_cast<const uint2*>(p) + v);
  o[0] = __uint_as_float(t.x << 16);
  o[1] = __uint_as_float(t.x & 0xFFFF0000u);
  o[2] = __uint_as_float(t.y << 16);
  o[3] = __uint_as_float(t.y & 0xFFFF0000u);
}

__device__ __forceinline__ void store4(float* p, int64_t v, const float (&o)[4]) {
  st_stream(reinterpret_cast<float4*>(p) + v, make_float4(o[0], o[1], o[2], o[3]));
}

// Round-to-nearest-even from the compute type (reading Z9).
__device__ __forceinline__ uint32_t bf16_bits(float x) {
  return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(x));
}
__device__ __forceinline__ uint32_t bf16_bits(double x) {
  return (uint32_t)__bfloat16_as_ushort(__double2bfloat16(x));
}

// ---- scalar element access (tails, unaligned leaf edges)
__device__ __forceinline__ float load1(const float* p, int64_t i) { return __ldcs(p + i); }
__device__ __forceinline__ float load1(const bf16* p, int64_t i) {
  return __uint_as_float(((uint32_t)__bfloat16_as_ushort(p[i])) << 16);
}

template <class CT>
__device__ __forceinline__ void store1(float* p, int64_t i, CT x) { __stcs(p + i, (float)x); }
template <class CT>
__device__ __forceinline__ void store1(bf16* p, int64_t i, CT x) {
  p[i] = __ushort_as_bfloat16((unsigned short)bf16_bits(x));
}

template <class CT>
__device__ __forceinline__ void store4c(float* p, int64_t v, const CT (&o)[4]) {
  const float f[4] = {(float)o[0], (float)o[1], (float)o[2], (float)o[3]};
  store4(p, v, f);
}
template <class CT>
__device__ __forceinline__ void store4c(bf16* p, int64_t v, const CT (&o)[4]) {
  uint2 t;
  t.x = bf16_bits(o[0]) | (bf16_bits(o[1]) << 16);
  t.y = bf16_bits(o[2]) | (bf16_bits(o[3]) << 16);
  st_stream(reinterpret_cast<uint2*>(p) + v, t);
}

// ---- cp.async (LDGSTS): global -> shared without staging in registers
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

}  // namespace dopt
