// Generic ADER-DG kernels (any order N, any quantity count P, fp64) used for the
// viscoelastic model (P = 27, reading R14; row A9 of SURVEY §8).  The global matrices are
// CSR arrays in device memory, the per-element coefficients use fixed sparsity patterns
// (star matrices: 3 columns per row; viscoelastic source E: 9; flux solvers: the 9
// elastic columns, since the Riemann state depends on the elastic quantities only).
//
// Layouts (element-major, canonical DOF layout = the ABI layout):
//   Q        [e][p][k]           traces  [e][face][m][q<9]
//   star     [e][c][p][3]        src     [e][p][9]
//   aplus/-  [e][face][p][9]     nb, jh  [e][4]
// One CTA handles kTE elements; every phase is a loop over (row, quantity, element) outputs
// with the contraction over a CSR row of the global matrix.
#include <cuda_runtime.h>

#include <cstdint>

#include "generic.h"

namespace ydg {
namespace gen {

constexpr int kTE = 4;  // elements per CTA

__constant__ int c_ecols[27][9];   // source-term column pattern of each row
__constant__ int c_scols[27][3];   // star-matrix column pattern of each row

struct Csr {
  const int* ptr;
  const int* col;
  const double* val;
};

__device__ __forceinline__ int idx3(int k, int p, int e, int P) { return (k * P + p) * kTE + e; }

__global__ void __launch_bounds__(256) gen_local(const GenParams prm) {
  extern __shared__ double sm[];
  const int B = prm.B, P = prm.P, Bt = prm.Bt;
  const int SZ = B * P * kTE;
  double* D = sm;
  double* Dn = D + SZ;
  double* I = Dn + SZ;
  double* X = I + SZ;  // [3][B][P][kTE]; later: traces / flux staging
  const int64_t e0 = prm.e0 + static_cast<int64_t>(blockIdx.x) * kTE;
  const int64_t left = prm.e0 + prm.n - e0;
  const int ne = static_cast<int>(left < kTE ? left : kTE);
  const Csr Kt{prm.kt_ptr, prm.kt_col, prm.kt_val}, Kh{prm.kh_ptr, prm.kh_col, prm.kh_val};
  const Csr Rt{prm.rt_ptr, prm.rt_col, prm.rt_val}, R{prm.r_ptr, prm.r_col, prm.r_val};
  // load Q, I = dt Q
  for (int i = threadIdx.x; i < SZ; i += blockDim.x) {
    const int e = i % kTE, kp = i / kTE, p = kp % P, k = kp / P;
    const double q = e < ne ? prm.Q[((e0 + e) * P + p) * B + k] : 0.0;
    D[i] = q;
    I[i] = prm.dt * q;
  }
  __syncthreads();
  auto star = [&](int e, int c, int p, int j) -> double {
    return e < ne ? prm.star[(((e0 + e) * 3 + c) * P + p) * 3 + j] : 0.0;
  };
  auto srcv = [&](int e, int p, int j) -> double {
    return (prm.src && e < ne) ? prm.src[((e0 + e) * P + p) * 9 + j] : 0.0;
  };
  // X^c = Dsrc A*^cT (all rows)
  auto make_x = [&](const double* Dsrc) {
    for (int i = threadIdx.x; i < 3 * SZ; i += blockDim.x) {
      const int c = i / SZ, r = i % SZ;
      const int e = r % kTE, kp = r / kTE, p = kp % P, l = kp / P;
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < 3; ++j) s = fma(star(e, c, p, j), Dsrc[idx3(l, c_scols[p][j], e, P)], s);
      X[i] = s;
    }
  };
  for (int d = 0; d < prm.N; ++d) {
    make_x(D);
    __syncthreads();
    const double sc = prm.scal[d], ic = prm.scal[prm.N + d];
    for (int i = threadIdx.x; i < SZ; i += blockDim.x) {
      const int e = i % kTE, kp = i / kTE, p = kp % P, k = kp / P;
      double s = 0.0;
      for (int c = 0; c < 3; ++c) {
        const int row = c * B + k;
        for (int t = Kt.ptr[row]; t < Kt.ptr[row + 1]; ++t) s = fma(Kt.val[t], X[c * SZ + idx3(Kt.col[t], p, e, P)], s);
      }
      if (prm.src)
        for (int j = 0; j < 9; ++j) s = fma(srcv(e, p, j), D[idx3(k, c_ecols[p][j], e, P)], s);
      const double v = sc * s;  // scaled derivative Dhat^{d+1} (reading R12)
      Dn[i] = v;
      I[i] = fma(ic, v, I[i]);
    }
    __syncthreads();
    double* t = D;
    D = Dn;
    Dn = t;
  }
  // volume: Q += sum_c Khat^c (I A*^cT) + I E^T
  make_x(I);
  __syncthreads();
  double* U = Dn;  // accumulated update [B][P][kTE]
  for (int i = threadIdx.x; i < SZ; i += blockDim.x) {
    const int e = i % kTE, kp = i / kTE, p = kp % P, k = kp / P;
    double s = 0.0;
    for (int c = 0; c < 3; ++c) {
      const int row = c * B + k;
      for (int t = Kh.ptr[row]; t < Kh.ptr[row + 1]; ++t) s = fma(Kh.val[t], X[c * SZ + idx3(Kh.col[t], p, e, P)], s);
    }
    if (prm.src)
      for (int j = 0; j < 9; ++j) s = fma(srcv(e, p, j), I[idx3(k, c_ecols[p][j], e, P)], s);
    U[i] = s;
  }
  __syncthreads();
  // traces T_i[m][q] = sum_l R^i[l][m] I[l][q], q < 9  -> X region [4][Bt][9][kTE] and global
  const int TS = Bt * 9 * kTE;
  for (int i = threadIdx.x; i < 4 * TS; i += blockDim.x) {
    const int f = i / TS, r = i % TS;
    const int e = r % kTE, mq = r / kTE, q = mq % 9, m = mq / 9;
    const int row = f * Bt + m;
    double s = 0.0;
    for (int t = Rt.ptr[row]; t < Rt.ptr[row + 1]; ++t) s = fma(Rt.val[t], I[idx3(Rt.col[t], q, e, P)], s);
    X[i] = s;
    if (e < ne) prm.traces[(((e0 + e) * 4 + f) * Bt + m) * 9 + q] = s;
  }
  __syncthreads();
  // local flux: Y_i[m][p] = sum_j A+_i[p][j] T_i[m][j]  -> X + 4 TS region [4][Bt][P][kTE]
  double* Y = X + 4 * TS;
  const int YS = Bt * P * kTE;
  for (int i = threadIdx.x; i < 4 * YS; i += blockDim.x) {
    const int f = i / YS, r = i % YS;
    const int e = r % kTE, mp = r / kTE, p = mp % P, m = mp / P;
    double s = 0.0;
    if (e < ne)
      for (int j = 0; j < 9; ++j) s = fma(prm.aplus[(((e0 + e) * 4 + f) * P + p) * 9 + j], X[f * TS + (m * 9 + j) * kTE + e], s);
    Y[i] = s;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < SZ; i += blockDim.x) {
    const int e = i % kTE, kp = i / kTE, p = kp % P, k = kp / P;
    double s = U[i];
    for (int f = 0; f < 4; ++f) {
      const int row = f * B + k;
      for (int t = R.ptr[row]; t < R.ptr[row + 1]; ++t) s = fma(R.val[t], Y[f * YS + (R.col[t] * P + p) * kTE + e], s);
    }
    if (e < ne) prm.Q[((e0 + e) * P + p) * B + k] += s;
  }
}

__global__ void __launch_bounds__(256) gen_neigh(const GenParams prm) {
  extern __shared__ double sm[];
  const int B = prm.B, P = prm.P, Bt = prm.Bt;
  const int64_t e0 = prm.e0 + static_cast<int64_t>(blockIdx.x) * kTE;
  const int64_t left = prm.e0 + prm.n - e0;
  const int ne = static_cast<int>(left < kTE ? left : kTE);
  const Csr R{prm.r_ptr, prm.r_col, prm.r_val}, Fh{prm.f_ptr, prm.f_col, prm.f_val};
  const int TS = Bt * 9 * kTE, YS = Bt * P * kTE;
  double* Z = sm;            // [4][Bt][9][kTE]
  double* Y = Z + 4 * TS;    // [4][Bt][P][kTE]
  // rotated neighbour traces z = f^h t
  for (int i = threadIdx.x; i < 4 * TS; i += blockDim.x) {
    const int f = i / TS, r = i % TS;
    const int e = r % kTE, mq = r / kTE, q = mq % 9, m = mq / 9;
    double s = 0.0;
    if (e < ne) {
      const int64_t nbe = prm.nb[(e0 + e) * 4 + f];
      const int jh = prm.jh[(e0 + e) * 4 + f];
      const int j = jh & 3, h = jh >> 2;
      const double* src = prm.traces + ((nbe * 4 + j) * Bt) * 9 + q;
      const int row = h * Bt + m;
      for (int t = Fh.ptr[row]; t < Fh.ptr[row + 1]; ++t) s = fma(Fh.val[t], src[Fh.col[t] * 9], s);
    }
    Z[i] = s;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4 * YS; i += blockDim.x) {
    const int f = i / YS, r = i % YS;
    const int e = r % kTE, mp = r / kTE, p = mp % P, m = mp / P;
    double s = 0.0;
    if (e < ne)
      for (int j = 0; j < 9; ++j) s = fma(prm.aminus[(((e0 + e) * 4 + f) * P + p) * 9 + j], Z[f * TS + (m * 9 + j) * kTE + e], s);
    Y[i] = s;
  }
  __syncthreads();
  const int SZ = B * P * kTE;
  for (int i = threadIdx.x; i < SZ; i += blockDim.x) {
    const int e = i % kTE, kp = i / kTE, p = kp % P, k = kp / P;
    double s = 0.0;
    for (int f = 0; f < 4; ++f) {
      const int row = f * B + k;
      for (int t = R.ptr[row]; t < R.ptr[row + 1]; ++t) s = fma(R.val[t], Y[f * YS + (R.col[t] * P + p) * kTE + e], s);
    }
    if (e < ne) prm.Q[((e0 + e) * P + p) * B + k] += s;
  }
}

}  // namespace gen

size_t gen_local_smem(int B, int Bt, int P) {
  const size_t SZ = static_cast<size_t>(B) * P * gen::kTE;
  const size_t extra = static_cast<size_t>(4) * Bt * 9 * gen::kTE + static_cast<size_t>(4) * Bt * P * gen::kTE;
  return (3 * SZ + (3 * SZ > extra ? 3 * SZ : extra)) * sizeof(double);
}
size_t gen_neigh_smem(int Bt, int P) {
  return (static_cast<size_t>(4) * Bt * 9 * gen::kTE + static_cast<size_t>(4) * Bt * P * gen::kTE) * sizeof(double);
}

cudaError_t gen_configure(int B, int Bt, int P, const int (*ecols)[9], const int (*scols)[3]) {
  cudaError_t e = cudaMemcpyToSymbol(gen::c_ecols, ecols, sizeof(int) * 27 * 9);
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(gen::c_scols, scols, sizeof(int) * 27 * 3);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(gen::gen_local, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(gen_local_smem(B, Bt, P)));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(gen::gen_neigh, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(gen_neigh_smem(Bt, P)));
  return e;
}

cudaError_t gen_launch(const GenParams& p, bool local, cudaStream_t s) {
  const int64_t blocks = (p.n + gen::kTE - 1) / gen::kTE;
  if (blocks <= 0) return cudaSuccess;
  if (local)
    gen::gen_local<<<static_cast<unsigned>(blocks), 256, gen_local_smem(p.B, p.Bt, p.P), s>>>(p);
  else
    gen::gen_neigh<<<static_cast<unsigned>(blocks), 256, gen_neigh_smem(p.Bt, p.P), s>>>(p);
  return cudaGetLastError();
}

int gen_tile_elems() { return gen::kTE; }

}  // namespace ydg
