// CUDA kernels of the ADER-DG element update for sm_100a (elastic, P = 9).
//
// Two launches per time step:
//   ader_local : CK recursion + time integral, volume,
//                face traces R^iT I
//   ader_neigh : local + neighbour flux R^i (T A+^T + (f^h T^nb) A-^T), one lift per face
//                (chain order P:1396)
// Thread = (element, quantity column); warp = 32 elements (a tile) x one column; CTA =
// the 9 columns of one tile.  Each nonzero of the global matrices is one FMA with a
// compile-time constant (generated/ydg_gen_N*.cuh); the per-element 9x9 mixing goes
// through shared memory laid out [row][quantity][lane] (conflict-free).
#include "kernels.cuh"

#include <algorithm>

namespace ydg {

// per-order kernel entry points (generated/kernels_N*.cu)
const void* local_fn_N1(int eb);
const void* neigh_fn_N1(int eb);
size_t local_smem_N1(int eb);
size_t neigh_smem_N1(int eb);
const void* local_fn_N2(int eb);
const void* neigh_fn_N2(int eb);
size_t local_smem_N2(int eb);
size_t neigh_smem_N2(int eb);
const void* local_fn_N3(int eb);
const void* neigh_fn_N3(int eb);
size_t local_smem_N3(int eb);
size_t neigh_smem_N3(int eb);
const void* local_fn_N4(int eb);
const void* neigh_fn_N4(int eb);
size_t local_smem_N4(int eb);
size_t neigh_smem_N4(int eb);
const void* local_fn_N5(int eb);
const void* neigh_fn_N5(int eb);
size_t local_smem_N5(int eb);
size_t neigh_smem_N5(int eb);
const void* local_fn_N6(int eb);
const void* neigh_fn_N6(int eb);
size_t local_smem_N6(int eb);
size_t neigh_smem_N6(int eb);
const void* fused_fn_N1();
size_t fused_smem_N1();
const void* fused_fn_N2();
size_t fused_smem_N2();
const void* fused_fn_N3();
size_t fused_smem_N3();
const void* fused_fn_N4();
size_t fused_smem_N4();
const void* fused_fn_N5();
size_t fused_smem_N5();
const void* fused_fn_N6();
size_t fused_smem_N6();

namespace {

constexpr int kP = 9;
constexpr int kRS = kP * kLanes;

// canonical [e][p][k] <-> tiled [tile][k][p][L] (L = 16 for fp64, 32 for fp32)
template <typename T>
__global__ void to_tiled_kernel(int P, int B, int L, const T* __restrict__ canon, T* __restrict__ tiled,
                                int64_t first, int64_t count, const int32_t* __restrict__ slot_of) {
  const int64_t n = count * P * B;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t el = i / (P * B);
    const int r = static_cast<int>(i - el * P * B);
    const int p = r / B, k = r - p * B;
    const int64_t e = slot_of ? slot_of[first + el] : first + el;
    tiled[((e / L) * B + k) * P * L + p * L + (e % L)] = canon[i];
  }
}
template <typename T>
__global__ void to_canonical_kernel(int P, int B, int L, const T* __restrict__ tiled, T* __restrict__ canon,
                                    int64_t first, int64_t count, const int32_t* __restrict__ slot_of) {
  const int64_t n = count * P * B;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t el = i / (P * B);
    const int r = static_cast<int>(i - el * P * B);
    const int p = r / B, k = r - p * B;
    const int64_t e = slot_of ? slot_of[first + el] : first + el;
    canon[i] = tiled[((e / L) * B + k) * P * L + p * L + (e % L)];
  }
}

// LTS trace bookkeeping: for every entry k, over the 4 faces of element slots: mode 0:
// dst = a; mode 1: dst = a - b; mode 2: dst += a.  Traces layout [tile][face][lane][TS].
__global__ void trace_combine_kernel(double* __restrict__ tr, const int64_t* __restrict__ lst, int64_t n, int TS,
                                     int L, int mode) {
  const int64_t total = n * 4 * TS;
  auto at = [&](int64_t s, int F, int v) { return (((s / L) * 4 + F) * L + (s % L)) * (int64_t)TS + v; };
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / (4 * TS);
    const int F = static_cast<int>((i / TS) % 4), v = static_cast<int>(i % TS);
    const int64_t d = lst[3 * k], a = lst[3 * k + 1], b = lst[3 * k + 2];
    const double va = tr[at(a, F, v)];
    if (mode == 0) tr[at(d, F, v)] = va;
    else if (mode == 1) tr[at(d, F, v)] = va - tr[at(b, F, v)];
    else tr[at(d, F, v)] += va;
  }
}

const void* pick_local(int N, int eb) {
  switch (N) {
    case 1: return local_fn_N1(eb);
    case 2: return local_fn_N2(eb);
    case 3: return local_fn_N3(eb);
    case 4: return local_fn_N4(eb);
    case 5: return local_fn_N5(eb);
    case 6: return local_fn_N6(eb);
  }
  return nullptr;
}
const void* pick_neigh(int N, int eb) {
  switch (N) {
    case 1: return neigh_fn_N1(eb);
    case 2: return neigh_fn_N2(eb);
    case 3: return neigh_fn_N3(eb);
    case 4: return neigh_fn_N4(eb);
    case 5: return neigh_fn_N5(eb);
    case 6: return neigh_fn_N6(eb);
  }
  return nullptr;
}
// fp64 tensor-core kernels: kDmWarps warps (dmma_impl.cuh kW); fp32 sparse kernels: 9 warps
int block_threads(int elem_bytes) { return elem_bytes == 8 ? kDmWarps * 32 * kLocalGroups : kP * kLanes; }
// fp64 flux kernel: 3 warps per CTA (8-element halves of the 16-element tiles)
int flux_threads(int elem_bytes) { return elem_bytes == 8 ? 3 * 32 * kFluxGroups : kP * kLanes; }
int nB(int N) { return (N + 1) * (N + 2) * (N + 3) / 6; }
int nBt(int N) { return (N + 1) * (N + 2) / 2; }

}  // namespace

size_t sparse_local_smem(int N, int eb) { return static_cast<size_t>(nB(N)) * kRS * eb; }
size_t sparse_neigh_smem(int N, int eb) { return static_cast<size_t>(6 * nBt(N)) * kRS * eb; }

size_t local_smem_bytes(int N, int eb) {
  switch (N) {
    case 1: return local_smem_N1(eb);
    case 2: return local_smem_N2(eb);
    case 3: return local_smem_N3(eb);
    case 4: return local_smem_N4(eb);
    case 5: return local_smem_N5(eb);
    case 6: return local_smem_N6(eb);
  }
  return 0;
}
size_t neigh_smem_bytes(int N, int eb) {
  switch (N) {
    case 1: return neigh_smem_N1(eb);
    case 2: return neigh_smem_N2(eb);
    case 3: return neigh_smem_N3(eb);
    case 4: return neigh_smem_N4(eb);
    case 5: return neigh_smem_N5(eb);
    case 6: return neigh_smem_N6(eb);
  }
  return 0;
}

const void* pick_fused(int N) {
  switch (N) {
    case 1: return fused_fn_N1();
    case 2: return fused_fn_N2();
    case 3: return fused_fn_N3();
    case 4: return fused_fn_N4();
    case 5: return fused_fn_N5();
    case 6: return fused_fn_N6();
  }
  return nullptr;
}
size_t fused_smem_bytes(int N) {
  switch (N) {
    case 1: return fused_smem_N1();
    case 2: return fused_smem_N2();
    case 3: return fused_smem_N3();
    case 4: return fused_smem_N4();
    case 5: return fused_smem_N5();
    case 6: return fused_smem_N6();
  }
  return 0;
}

cudaError_t configure_kernels(int N, int eb) {
  const void* fl = pick_local(N, eb);
  const void* fn = pick_neigh(N, eb);
  if (!fl || !fn) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(fl, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(local_smem_bytes(N, eb)));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(neigh_smem_bytes(N, eb)));
  // all of the unified L1 / shared memory as shared memory (two fp64 CTAs per SM)
  if (e == cudaSuccess) e = cudaFuncSetAttribute(fl, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e == cudaSuccess && eb == 8) {
    const void* ff = pick_fused(N);
    e = cudaFuncSetAttribute(ff, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(fused_smem_bytes(N)));
    if (e == cudaSuccess) e = cudaFuncSetAttribute(ff, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  }
  return e;
}

// grid counts work groups (virtual CTAs) as for the local kernel
cudaError_t launch_fused(int N, const StepParams<double>& p, int grid, cudaStream_t s) {
  const void* f = pick_fused(N);
  if (!f) return cudaErrorInvalidValue;
  void* args[] = {const_cast<StepParams<double>*>(&p)};
  const int ctas = (grid + kLocalGroups - 1) / kLocalGroups;
  return cudaLaunchKernel(f, dim3(ctas), dim3(block_threads(8)), args, fused_smem_bytes(N), s);
}

template <typename T>
cudaError_t launch_local(int N, const StepParams<T>& p, int grid, cudaStream_t s) {
  const void* f = pick_local(N, sizeof(T));
  if (!f) return cudaErrorInvalidValue;
  void* args[] = {const_cast<StepParams<T>*>(&p)};
  // fp64: grid counts work groups (virtual CTAs); kLocalGroups of them share one CTA
  const int ctas = sizeof(T) == 8 ? (grid + kLocalGroups - 1) / kLocalGroups : grid;
  return cudaLaunchKernel(f, dim3(ctas), dim3(block_threads(sizeof(T))), args, local_smem_bytes(N, sizeof(T)), s);
}
template <typename T>
cudaError_t launch_neigh(int N, const StepParams<T>& p, int grid, cudaStream_t s) {
  const void* f = pick_neigh(N, sizeof(T));
  if (!f) return cudaErrorInvalidValue;
  void* args[] = {const_cast<StepParams<T>*>(&p)};
  // fp64: grid counts 3-warp groups (virtual CTAs); kFluxGroups of them share one CTA
  const int ctas = sizeof(T) == 8 ? (grid + kFluxGroups - 1) / kFluxGroups : grid;
  return cudaLaunchKernel(f, dim3(ctas), dim3(flux_threads(sizeof(T))), args, neigh_smem_bytes(N, sizeof(T)), s);
}
// max |Q| over the owned elements (diagnostic): L > 0 = tiled layout
// [tile][k][p][L] (element = tile * L + lane), L = 0 = canonical [e][p][k]; a non-finite
// value sets *bad.  out holds the bit pattern of a non-negative double (ordered like the
// value, so atomicMax on the bits is a max on the values).
template <typename T>
__global__ void maxabs_kernel(const T* Q, int64_t n, int64_t per_tile, int L, int64_t per_elem, int64_t nlocal,
                              unsigned long long* out, int* bad) {
  double m = 0.0;
  int b = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t e = L > 0 ? (i / per_tile) * L + i % L : i / per_elem;
    if (e >= nlocal) continue;
    const double v = static_cast<double>(Q[i]);
    if (!isfinite(v)) b = 1;
    else m = fmax(m, fabs(v));
  }
  for (int o = 16; o > 0; o >>= 1) {
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    b |= __shfl_xor_sync(0xffffffffu, b, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(m)));
    if (b) atomicOr(bad, 1);
  }
}
template <typename T>
cudaError_t launch_maxabs(const T* Q, int64_t n, int64_t per_tile, int L, int64_t per_elem, int64_t nlocal,
                          unsigned long long* out, int* bad, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  maxabs_kernel<T><<<148 * 8, 256, 0, s>>>(Q, n, per_tile, L, per_elem, nlocal, out, bad);
  return cudaGetLastError();
}
template cudaError_t launch_maxabs<double>(const double*, int64_t, int64_t, int, int64_t, int64_t, unsigned long long*,
                                           int*, cudaStream_t);
template cudaError_t launch_maxabs<float>(const float*, int64_t, int64_t, int, int64_t, int64_t, unsigned long long*,
                                          int*, cudaStream_t);

cudaError_t launch_trace_combine(double* traces, const int64_t* lst, int64_t n, int TS, int L, int mode,
                                 cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  trace_combine_kernel<<<148 * 4, 256, 0, s>>>(traces, lst, n, TS, L, mode);
  return cudaGetLastError();
}
template <typename T>
cudaError_t launch_to_tiled(int P, int B, int L, const T* canon, T* tiled, int64_t first, int64_t count,
                            const int32_t* slot_of, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  to_tiled_kernel<T><<<148 * 8, 256, 0, s>>>(P, B, L, canon, tiled, first, count, slot_of);
  return cudaGetLastError();
}
template <typename T>
cudaError_t launch_to_canonical(int P, int B, int L, const T* tiled, T* canon, int64_t first,
                                int64_t count, const int32_t* slot_of, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  to_canonical_kernel<T><<<148 * 8, 256, 0, s>>>(P, B, L, tiled, canon, first, count, slot_of);
  return cudaGetLastError();
}

template cudaError_t launch_local<double>(int, const StepParams<double>&, int, cudaStream_t);
template cudaError_t launch_local<float>(int, const StepParams<float>&, int, cudaStream_t);
template cudaError_t launch_neigh<double>(int, const StepParams<double>&, int, cudaStream_t);
template cudaError_t launch_neigh<float>(int, const StepParams<float>&, int, cudaStream_t);
template cudaError_t launch_to_tiled<double>(int, int, int, const double*, double*, int64_t, int64_t, const int32_t*, cudaStream_t);
template cudaError_t launch_to_tiled<float>(int, int, int, const float*, float*, int64_t, int64_t, const int32_t*, cudaStream_t);
template cudaError_t launch_to_canonical<double>(int, int, int, const double*, double*, int64_t, int64_t, const int32_t*, cudaStream_t);
template cudaError_t launch_to_canonical<float>(int, int, int, const float*, float*, int64_t, int64_t, const int32_t*, cudaStream_t);

}  // namespace ydg
