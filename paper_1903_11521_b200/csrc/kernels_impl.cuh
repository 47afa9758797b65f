// Templated ADER-DG kernels (elastic, P = 9); instantiated per order in
// generated/kernels_N*.cu so that the large unrolled bodies compile in parallel.
//
// Thread = (element lane, quantity column p); warp = one column of a 32-element tile; CTA =
// the 9 columns of one tile (9 warps: 3 on one SM sub-partition, so <= 168 registers per
// thread).  Every phase keeps at most one B-long accumulator column in registers; the
// cross-column mixing by the star matrices and flux solvers reads shared memory laid
// out [row][q][lane] (each warp load hits 32 consecutive words: conflict-free).
#pragma once
#include "kernels.cuh"

namespace ydg {
template <int N>
struct Gen;
}

namespace ydg {
namespace kimpl {

constexpr int kP = 9;
constexpr int kRS = kP * kLanes;  // row stride of [row][q][lane]

// YDG_FQPF: the tile's Q rows -> L2 ahead of its read-modify-write (the staging read of the
// local kernel was ~100 us earlier and has left the L2; the neighbour kernel reads Q last)
#ifndef YDG_FQPF
#define YDG_FQPF 1  // measured (c2): ader_neigh 23.40 -> 23.10 ms, ader_local unchanged
#endif
__device__ __forceinline__ void q_prefetch_l2(const void* p, unsigned bytes) {
  if constexpr (YDG_FQPF != 0)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// 3-column pattern of star-matrix row p (same table as setup.cpp star_cols)
static __constant__ int c_star_cols[9][3] = {{6, 7, 8}, {6, 7, 8}, {6, 7, 8}, {6, 7, 7}, {7, 8, 8},
                                             {6, 8, 8}, {0, 3, 5}, {3, 1, 4}, {5, 4, 2}};

template <typename T>
__device__ __forceinline__ void load_flux_row(const T* base, int64_t tile, int F, int p, int lane,
                                              T (&arow)[kP]) {
  const T* A = base + ((tile * 4 + F) * kP + p) * kP * kLanes + lane;
#pragma unroll
  for (int q = 0; q < kP; ++q) arow[q] = A[q * kLanes];
}

template <typename T, int B>
__device__ __forceinline__ void add_to_q(T* Qt, const T (&acc)[B]) {
#pragma unroll
  for (int k0 = 0; k0 < B; k0 += 8) {
    asm volatile("" ::: "memory");  // at most 8 loads of Q in flight
#pragma unroll
    for (int k = k0; k < (k0 + 8 < B ? k0 + 8 : B); ++k) Qt[k * kRS] += acc[k];
  }
}

// Local part of the update: CK recursion + time integral, volume
// and the traces T_i = R^iT I (stored for the flux kernel).  Shared memory:
// S [B][9][32].
template <int N, typename T>
__global__ void __launch_bounds__(kP * kLanes, 1) ader_local(const StepParams<T> prm) {
  using G = Gen<N>;
  constexpr int B = G::B, Bt = G::Bt;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* S = reinterpret_cast<T*>(smem_raw);  // [B][9][32]
  const int lane = threadIdx.x & 31, p = threadIdx.x >> 5;
  const int c0 = c_star_cols[p][0], c1 = c_star_cols[p][1], c2 = c_star_cols[p][2];
  const int own = p * kLanes + lane;
  for (int64_t it = blockIdx.x; it < prm.ntiles; it += gridDim.x) {
    const int64_t tile = prm.tile0 + it;
    T* Qt = prm.Q + tile * B * kRS + own;
#pragma unroll 8
    for (int k = 0; k < B; ++k) S[k * kRS + own] = Qt[k * kRS];
    T a[9];
    const T* st = prm.star + (tile * 3 * kP) * 3 * kLanes + lane;
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int j = 0; j < 3; ++j) a[3 * c + j] = st[((c * kP + p) * 3 + j) * kLanes];
    __syncthreads();
    {
      T I[G::Bv];
      G::template ck<T>(S + c0 * kLanes + lane, S + c1 * kLanes + lane, S + c2 * kLanes + lane,
                        S + own, a, I, prm.scal, prm.dt);
      // ck ends with a barrier; the own column now receives the time integral: rows < Bv
      // from I, rows >= Bv are dt * Q (still in shared memory)
#pragma unroll
      for (int k = 0; k < G::Bv; ++k) S[k * kRS + own] = I[k];
#pragma unroll 8
      for (int k = G::Bv; k < B; ++k) S[k * kRS + own] = prm.dt * S[k * kRS + own];
    }
    __syncthreads();
    if (threadIdx.x == 0) q_prefetch_l2(prm.Q + tile * B * kRS, B * kRS * sizeof(T));
    {
      T acc[B];
#pragma unroll
      for (int k = 0; k < B; ++k) acc[k] = T(0);
      G::template volume<T>(S + c0 * kLanes + lane, S + c1 * kLanes + lane, S + c2 * kLanes + lane, a,
                            acc);
      add_to_q(Qt, acc);
    }
    // traces of the time integral on the four faces (own column), stored for the flux
    // kernel, tiled trace layout [tile][face][m][q][32]; both flux terms are applied there
    // (one lift per face, as on the fp64 path)
    T* tr = prm.traces + tile * 4 * Bt * kRS + p * kLanes + lane;
    {
      T ta[Bt], tb[Bt];
      G::template trace<0, T>(S + own, ta);
      G::template trace<1, T>(S + own, tb);
#pragma unroll
      for (int m = 0; m < Bt; ++m) {
        tr[(0 * Bt + m) * kRS] = ta[m];
        tr[(1 * Bt + m) * kRS] = tb[m];
      }
      G::template trace<2, T>(S + own, ta);
      G::template trace<3, T>(S + own, tb);
#pragma unroll
      for (int m = 0; m < Bt; ++m) {
        tr[(2 * Bt + m) * kRS] = ta[m];
        tr[(3 * Bt + m) * kRS] = tb[m];
      }
    }
    __syncthreads();  // before the next tile overwrites S
  }
}

// Flux of face F on the own column p (P:1341-1342 with one lift per face, reading R22):
//   y_m = sum_q T_i[m][q] A+_i[p][q] + sum_q Z_i[m][q] A-_i[p][q]
// O = the tile's own trace rows of the face (staged in shared memory, [m][q][32]), Z = the
// rotated neighbour trace (replaced by y).
template <int Bt, typename T>
__device__ __forceinline__ void mix_flux(T* Z, const T* O, const T* ap, const T* am, int64_t tile, int F, int p,
                                         int lane) {
  T y[Bt];
  {
    T rp[kP], rm[kP];
    load_flux_row(ap, tile, F, p, lane, rp);
    load_flux_row(am, tile, F, p, lane, rm);
#pragma unroll
    for (int m = 0; m < Bt; ++m) {
      asm volatile("" ::: "memory");  // one row of loads in flight: bounded register pressure
      const T* row = Z + m * kRS + lane;
      const T* orow = O + m * kRS + lane;
      T s = T(0), u = T(0);
#pragma unroll
      for (int q = 0; q < kP; ++q) s = fma(row[q * kLanes], rm[q], s);
#pragma unroll
      for (int q = 0; q < kP; ++q) u = fma(orow[q * kLanes], rp[q], u);
      y[m] = s + u;
    }
  }
  __syncthreads();  // every column of Z and O has been read
#pragma unroll
  for (int m = 0; m < Bt; ++m) Z[m * kRS + p * kLanes + lane] = y[m];
}

// the tile's own traces of face F -> O (16-byte cp.async, one commit group)
template <int Bt, typename T>
__device__ __forceinline__ void own_copy(const T* traces, int64_t tile, int F, T* O) {
  constexpr int n = Bt * kRS * static_cast<int>(sizeof(T)) / 16;
  const char* src = reinterpret_cast<const char*>(traces + (tile * 4 + F) * Bt * kRS);
  char* dst = reinterpret_cast<char*>(O);
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst + 16 * i))),
                 "l"(src + 16 * i)
                 : "memory");
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int K>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(K) : "memory");
}

template <int N, typename T, int F>
__device__ __forceinline__ void neigh_gather(const StepParams<T>& prm, int64_t tile, int p, int lane,
                                            T* ZF) {
  using G = Gen<N>;
  constexpr int Bt = G::Bt;
  const int64_t slot = (tile * 4 + F) * kLanes + lane;
  const int64_t nbe = prm.nb[slot];
  const int jh = prm.jh[slot];
  const int j = jh & 3, h = jh >> 2;
  const T* src = prm.traces + (((nbe >> 5) * 4 + j) * Bt) * kRS + p * kLanes + (nbe & 31);
  T tn[Bt];
#pragma unroll
  for (int n = 0; n < Bt; ++n) tn[n] = src[n * kRS];
  T* dst = ZF + p * kLanes + lane;
  G::template rot<T>(h, tn, [&](int m, T z) { dst[m * kRS] = z; });
}

// Flux kernel (chain order P:1396) with one lift per face (reading R22):
//   Q += sum_i R^i ( T_i A+_i^T + (f^h_i T^nb_(j_i)) A-_i^T ).
// Shared memory: Z [4][Bt][9][32] (rotated neighbour traces, then the face fluxes), O
// [2][Bt][9][32] (the tile's own traces of two faces at a time).
template <int N, typename T>
__global__ void __launch_bounds__(kP * kLanes, 1) ader_neigh(const StepParams<T> prm) {
  using G = Gen<N>;
  constexpr int B = G::B, Bt = G::Bt;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Z = reinterpret_cast<T*>(smem_raw);
  const int lane = threadIdx.x & 31, p = threadIdx.x >> 5;
  const int own = p * kLanes + lane;
  for (int64_t it = blockIdx.x; it < prm.ntiles; it += gridDim.x) {
    const int64_t tile = prm.tile0 + it;
    if (threadIdx.x == 0) q_prefetch_l2(prm.Q + tile * B * kRS, B * kRS * sizeof(T));
    T* O0 = Z + 4 * Bt * kRS;
    T* O1 = O0 + Bt * kRS;
    own_copy<Bt>(prm.traces, tile, 0, O0);
    own_copy<Bt>(prm.traces, tile, 1, O1);
    neigh_gather<N, T, 0>(prm, tile, p, lane, Z + 0 * Bt * kRS);
    neigh_gather<N, T, 1>(prm, tile, p, lane, Z + 1 * Bt * kRS);
    neigh_gather<N, T, 2>(prm, tile, p, lane, Z + 2 * Bt * kRS);
    neigh_gather<N, T, 3>(prm, tile, p, lane, Z + 3 * Bt * kRS);
    cp_async_wait_group<0>();
    __syncthreads();  // rotated neighbour traces, own traces of faces 0, 1 in shared memory
    mix_flux<Bt>(Z + 0 * Bt * kRS, O0, prm.aplus, prm.aminus, tile, 0, p, lane);
    own_copy<Bt>(prm.traces, tile, 2, O0);
    mix_flux<Bt>(Z + 1 * Bt * kRS, O1, prm.aplus, prm.aminus, tile, 1, p, lane);
    own_copy<Bt>(prm.traces, tile, 3, O1);
    cp_async_wait_group<1>();
    __syncthreads();  // face 2's own traces
    mix_flux<Bt>(Z + 2 * Bt * kRS, O0, prm.aplus, prm.aminus, tile, 2, p, lane);
    cp_async_wait_group<0>();
    __syncthreads();  // face 3's own traces
    mix_flux<Bt>(Z + 3 * Bt * kRS, O1, prm.aplus, prm.aminus, tile, 3, p, lane);
    __syncthreads();
    T acc[B];
#pragma unroll
    for (int k = 0; k < B; ++k) acc[k] = T(0);
    G::template lift<0, T>(Z + 0 * Bt * kRS + own, acc);
    G::template lift<1, T>(Z + 1 * Bt * kRS + own, acc);
    G::template lift<2, T>(Z + 2 * Bt * kRS + own, acc);
    G::template lift<3, T>(Z + 3 * Bt * kRS + own, acc);
    add_to_q(prm.Q + tile * B * kRS + own, acc);
    __syncthreads();
  }
}

}  // namespace kimpl
}  // namespace ydg
