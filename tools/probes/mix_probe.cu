// Streaming ceiling by read/write mix: a kernel that reads NR fp32 arrays and
// writes NW (out_j = sum of inputs + j), float4 grid-stride, no other work.
// Grids: persistent (148 SMs x 3 blocks of 256, the optimizer kernels' shape)
// and full (one block per 256*U vectors). Back-to-back launches timed with
// CUDA events over rotating buffer sets (every launch reads HBM).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mix_probe mix_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int NR, int NW, int U>
__global__ void __launch_bounds__(256) mix(const float4* const* in, float4* const* out, long nv) {
  const long nt = (long)gridDim.x * blockDim.x;
  long v = (long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; v + (U - 1) * nt < nv; v += U * nt) {
    float4 x[U][NR];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int r = 0; r < NR; ++r) x[u][r] = __ldcs(in[r] + v + u * nt);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float4 s = x[u][0];
#pragma unroll
      for (int r = 1; r < NR; ++r) s.x += x[u][r].x, s.y += x[u][r].y, s.z += x[u][r].z, s.w += x[u][r].w;
#pragma unroll
      for (int w = 0; w < NW; ++w) __stcs(out[w] + v + u * nt, make_float4(s.x + w, s.y, s.z, s.w));
    }
  }
  for (; v < nv; v += nt) {
    float4 s = __ldcs(in[0] + v);
#pragma unroll
    for (int r = 1; r < NR; ++r) { float4 t = __ldcs(in[r] + v); s.x += t.x, s.y += t.y, s.z += t.z, s.w += t.w; }
#pragma unroll
    for (int w = 0; w < NW; ++w) __stcs(out[w] + v, make_float4(s.x + w, s.y, s.z, s.w));
  }
}

template <int NR, int NW, int U>
void run(long n, int sets, int reps, bool full) {
  const long nv = n / 4;
  float4 **din, **dout;
  cudaMalloc(&din, sizeof(float4*) * NR * sets);
  cudaMalloc(&dout, sizeof(float4*) * NW * sets);
  float4* hin[64]; float4* hout[64];
  for (int i = 0; i < NR * sets; ++i) { cudaMalloc(&hin[i], nv * 16); cudaMemset(hin[i], 0, nv * 16); }
  for (int i = 0; i < NW * sets; ++i) cudaMalloc(&hout[i], nv * 16);
  cudaMemcpy(din, hin, sizeof(float4*) * NR * sets, cudaMemcpyHostToDevice);
  cudaMemcpy(dout, hout, sizeof(float4*) * NW * sets, cudaMemcpyHostToDevice);
  const int grid = full ? (int)((nv + 256L * U - 1) / (256L * U)) : 148 * 3;
  for (int i = 0; i < 10; ++i) mix<NR, NW, U><<<grid, 256>>>(din + (i % sets) * NR, dout + (i % sets) * NW, nv);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) mix<NR, NW, U><<<grid, 256>>>(din + (i % sets) * NR, dout + (i % sets) * NW, nv);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double us = ms * 1e3 / reps, bytes = (double)n * 4 * (NR + NW);
  printf("{\"n\": %ld, \"reads\": %d, \"writes\": %d, \"U\": %d, \"grid\": \"%s\", \"us\": %.3f, \"gbs\": %.1f}\n",
         n, NR, NW, U, full ? "full" : "persistent", us, bytes / us * 1e-3);
  for (int i = 0; i < NR * sets; ++i) cudaFree(hin[i]);
  for (int i = 0; i < NW * sets; ++i) cudaFree(hout[i]);
  cudaFree(din); cudaFree(dout);
}

int main() {
  const long sizes[2] = {11689512L / 4 * 4, 1L << 28};
  for (int si = 0; si < 2; ++si) {
    const long n = sizes[si];
    const int sets = si == 0 ? 2 : 1, reps = si == 0 ? 200 : 10;
    for (int full = 0; full < 2; ++full) {
      run<1, 1, 4>(n, sets, reps, full);
      run<3, 3, 2>(n, sets, reps, full);
      run<6, 3, 2>(n, sets, reps, full);
      run<2, 1, 4>(n, sets, reps, full);
      run<6, 0 + 3, 1>(n, sets, reps, full);
      run<4, 0 + 4, 2>(n, sets, reps, full);
    }
  }
  return 0;
}
