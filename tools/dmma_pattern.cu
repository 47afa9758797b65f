// Micro-benchmark of the DMMA inner-loop pattern of dm_local (12 warps, 1 CTA/SM):
// per k-set, B fragments from shared memory (3 units), TPK A fragments from a global
// table (or shared memory), TPK x 3 DMMAs into MT x 3 accumulators.  Prints DMMA
// throughput as a fraction of the 16-cycle-per-SMSP peak.
#include <cstdio>
#include <cuda_runtime.h>

template <int MT, int TPK, int ASRC, int XC = 0>
__global__ void __launch_bounds__(384, 1) pat(const double* __restrict__ frags, int nfr, int ksets, double* out,
                                              long long* cyc) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 20000; i += 384) sm[i] = 1.0 + 1e-9 * i;
  __syncthreads();
  double acc[MT][3][2] = {};
  long long t0 = clock64();
  int tid = w;
  for (int ks = 0; ks < ksets; ++ks) {
    double bf[3];
    if (XC) {  // star chunk: 12 loads, 36 FP64 ops, 12 stores, syncwarp, B fragments from it
      double* xb = sm + 16000 + w * 288;
      __syncwarp();
      if ((lane >> 3) < 3) {
        double d[4][3];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int j = 0; j < 3; ++j) d[r][j] = sm[((ks * 4 + r) & 31) * 288 + ((j * 3 + (lane >> 3)) % 9) * 32 + (lane & 7) + 8 * (w & 3)];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 3; ++c)
            xb[((c * 3 + (lane >> 3)) * 4 + r) * 8 + (lane & 7)] =
                fma(1.0001 * c, d[r][2], fma(0.9999, d[r][1], 1.00001 * d[r][0]));
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 3; ++k) bf[k] = xb[((((ks % 3)) * 3 + k) * 4 + (lane & 3)) * 8 + (lane >> 2)];
    } else {
#pragma unroll
    for (int k = 0; k < 3; ++k) bf[k] = sm[(ks & 63) * 288 + k * 32 + (lane >> 2) + 8 * (w & 3)];
    }
#pragma unroll
    for (int t = 0; t < TPK; ++t) {
      double a;
      if (ASRC == 0) a = __ldg(frags + ((tid + t) % nfr) * 32 + lane);
      else a = sm[19000 - ((tid + t) & 31) * 32 + lane];
#pragma unroll
      for (int k = 0; k < 3; ++k)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[t % MT][k][0]), "+d"(acc[t % MT][k][1])
                     : "d"(a), "d"(bf[k]));
    }
    tid += TPK;
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int k = 0; k < 3; ++k) s += acc[m][k][0] + acc[m][k][1];
  out[blockIdx.x * 384 + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MT, int TPK, int ASRC, int XC = 0>
void run(const char* name, const double* fr, int nfr, double* out, long long* cyc) {
  const int ksets = 2000;
  cudaFuncSetAttribute(pat<MT, TPK, ASRC, XC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  pat<MT, TPK, ASRC, XC><<<148, 384, 200 * 1024>>>(fr, nfr, ksets, out, cyc);
  pat<MT, TPK, ASRC, XC><<<148, 384, 200 * 1024>>>(fr, nfr, ksets, out, cyc);
  cudaDeviceSynchronize();
  long long c[148];
  cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < 148; ++i) mean += c[i] / 148.0;
  // DMMAs per SMSP = 3 warps * ksets * TPK * 3; peak 1 per 16 cycles
  const double dmma = 3.0 * ksets * TPK * 3;
  printf("%-28s cycles %.0f  dmma/SMSP %.0f  frac of peak %.3f\n", name, mean, dmma, dmma * 16.0 / mean);
}

int main() {
  const int nfr = 460;
  double *fr, *out;
  long long* cyc;
  cudaMalloc(&fr, nfr * 32 * 8);
  cudaMemset(fr, 0, nfr * 32 * 8);
  cudaMalloc(&out, 148 * 384 * 8);
  cudaMalloc(&cyc, 148 * 8);
  run<5, 7, 0>("MT5 TPK7 A:global", fr, nfr, out, cyc);
  run<5, 7, 1>("MT5 TPK7 A:smem", fr, nfr, out, cyc);
  run<5, 20, 0>("MT5 TPK20 A:global", fr, nfr, out, cyc);
  run<5, 20, 1>("MT5 TPK20 A:smem", fr, nfr, out, cyc);
  run<8, 16, 1>("MT8 TPK16 A:smem", fr, nfr, out, cyc);
  run<2, 8, 1>("MT2 TPK8 A:smem", fr, nfr, out, cyc);
  run<5, 7, 0>("MT5 TPK7 A:global(small tbl)", fr, 40, out, cyc);
  run<5, 7, 1, 1>("MT5 TPK7 A:smem +xcalc", fr, nfr, out, cyc);
  run<5, 7, 0, 1>("MT5 TPK7 A:global +xcalc", fr, nfr, out, cyc);
  run<5, 14, 1, 1>("MT5 TPK14 A:smem +xcalc", fr, nfr, out, cyc);
  return 0;
}
