// Micro-benchmarks for the roofline denominators the ADER-DG path needs and
// MEASURED_PEAKS.json lacks: FP64 FMA (DFMA), FP64 tensor (DMMA 8x8x4),
// FP32 FMA, HBM read / copy.  Prints one JSON object on stdout.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks tools/peaks.cu
//
// Each compute test runs a short burst (best of 5) and a ~2 s sustained loop.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) dfma_kernel(double* out, int iters, double s) {
  double a[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double m = 0.999999, c = s;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int i = 0; i < kChains; ++i) a[i] = fma(a[i], m, c);
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) t += a[i];
  if (t == 12345.678) out[threadIdx.x] = t;
}

__global__ void __launch_bounds__(256) ffma_kernel(float* out, int iters, float s) {
  float a[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) a[i] = threadIdx.x * 1e-3f + i;
  const float m = 0.999999f, c = s;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int i = 0; i < kChains; ++i) a[i] = fmaf(a[i], m, c);
  }
  float t = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) t += a[i];
  if (t == 12345.678f) out[threadIdx.x] = t;
}

// DMMA m8n8k4: 8*8*4 = 256 FMA per warp-instruction.
__global__ void __launch_bounds__(256) dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int i = 0; i < 4; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) t += c[i][0] + c[i][1];
  if (t == 12345.678) out[threadIdx.x] = t;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = __ldcs(a + i);
}
__global__ void read_kernel(const double2* __restrict__ a, double* out, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  double s = 0;
  for (; i < n; i += st) { double2 v = __ldcs(a + i); s += v.x + v.y; }
  if (s == 12345.678) out[0] = s;
}

template <class F>
static void timed(F f, int reps, float* best, float* total) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  f(); CK(cudaDeviceSynchronize());
  *best = 1e30f; *total = 0;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0)); f(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    *best = std::min(*best, ms); *total += ms;
  }
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  const int sms = p.multiProcessorCount;
  double* dout; CK(cudaMalloc(&dout, 1 << 20));
  const int blocks = sms * 8, threads = 256;
  printf("{\"gpu\": \"%s\", \"sms\": %d", p.name, sms);
  // FP64 FMA
  {
    int iters = 2000;
    float best, tot;
    auto f = [&] { dfma_kernel<<<blocks, threads>>>(dout, iters, 1e-9); };
    timed(f, 5, &best, &tot);
    double fl = 2.0 * blocks * threads * (double)iters * 16 * kChains;
    printf(", \"fp64_fma_tflops\": %.2f", fl / best * 1e-9);
    int reps = std::max(1, (int)(2000.0 / best));
    timed(f, reps, &best, &tot);
    printf(", \"fp64_fma_tflops_sustained\": %.2f", fl * reps / tot * 1e-9);
  }
  // FP64 DMMA
  {
    int iters = 1000;
    float best, tot;
    auto f = [&] { dmma_kernel<<<blocks, threads>>>(dout, iters); };
    timed(f, 5, &best, &tot);
    double fl = 2.0 * 256 * (blocks * threads / 32) * (double)iters * 16 * 4;
    printf(", \"fp64_dmma_tflops\": %.2f", fl / best * 1e-9);
    int reps = std::max(1, (int)(2000.0 / best));
    timed(f, reps, &best, &tot);
    printf(", \"fp64_dmma_tflops_sustained\": %.2f", fl * reps / tot * 1e-9);
  }
  // FP32 FMA
  {
    int iters = 4000;
    float best, tot;
    auto f = [&] { ffma_kernel<<<blocks, threads>>>((float*)dout, iters, 1e-9f); };
    timed(f, 5, &best, &tot);
    double fl = 2.0 * blocks * threads * (double)iters * 16 * kChains;
    printf(", \"fp32_fma_tflops\": %.2f", fl / best * 1e-9);
    int reps = std::max(1, (int)(2000.0 / best));
    timed(f, reps, &best, &tot);
    printf(", \"fp32_fma_tflops_sustained\": %.2f", fl * reps / tot * 1e-9);
  }
  // HBM
  {
    size_t n = (size_t)1 << 28;  // 2^28 double2 = 4 GiB per buffer
    double2 *a, *b;
    CK(cudaMalloc(&a, n * sizeof(double2))); CK(cudaMalloc(&b, n * sizeof(double2)));
    CK(cudaMemset(a, 0, n * sizeof(double2)));
    float best, tot;
    timed([&] { copy_kernel<<<sms * 16, 512>>>(a, b, n); }, 10, &best, &tot);
    printf(", \"hbm_copy_gbs\": %.1f", 2.0 * n * sizeof(double2) / best * 1e-6);
    timed([&] { read_kernel<<<sms * 16, 512>>>(a, dout, n); }, 10, &best, &tot);
    printf(", \"hbm_read_gbs\": %.1f", 1.0 * n * sizeof(double2) / best * 1e-6);
    CK(cudaFree(a)); CK(cudaFree(b));
  }
  int clk = 0; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  printf(", \"sm_clock_max_mhz\": %.0f}\n", clk / 1000.0);
  return 0;
}
