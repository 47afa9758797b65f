// DMMA m8n8k4 (fp64) throughput on one B200 against the number of independent accumulator
// chains per warp and the number of warps per SM: does the dm_local shape (3 warps per
// sub-partition, 3..15 chains in flight per warp) reach the pipe peak, or is a dependent
// DMMA's latency exposed (the `wait` stall of the ncu profile)?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_chains tools/dmma_chains.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void chains(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[C][2];
#pragma unroll
  for (int i = 0; i < C; ++i) c[i][0] = c[i][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 24 / C; ++u)
#pragma unroll
      for (int i = 0; i < C; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < C; ++i) t += c[i][0] + c[i][1];
  if (t == 12345.678) out[threadIdx.x] = t;
}

template <int C>
static void run(int sms, int warps, double* d) {
  const int iters = 2000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  chains<C><<<sms, warps * 32>>>(d, 10);
  cudaEventRecord(e0);
  chains<C><<<sms, warps * 32>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 2.0 * 256 * 32 / 32 * (24 / C) * C * (double)iters * warps * sms;  // per-warp 256 FMA x 2
  printf("{\"chains\": %d, \"warps_per_sm\": %d, \"tflops\": %.2f}\n", C, warps, fl / (ms * 1e-3) * 1e-12);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 1 << 20);
  for (int w : {4, 8, 12, 16}) {
    run<1>(sms, w, d);
    run<2>(sms, w, d);
    run<3>(sms, w, d);
    run<4>(sms, w, d);
    run<6>(sms, w, d);
    run<8>(sms, w, d);
  }
  return 0;
}
