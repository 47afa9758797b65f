// Generic ADER-DG kernels (any order N, P = 9 or 27 quantities, fp64) used for the
// viscoelastic model (P = 27, reading R14; row A9 of SURVEY §8) and for N = 6 in fp64.  The
// global matrices are CSR arrays in device memory, the per-element coefficients use fixed
// sparsity patterns (star matrices: 3 columns per row; viscoelastic source E: 9; flux
// solvers: the 9 elastic columns, since the Riemann state depends on the elastic
// quantities only).
//
// Layouts (element-major, canonical DOF layout = the ABI layout):
//   Q        [e][p][k]           traces  [e][face][m][q<9]
//   star     [e][c][p][3]        src     [e][p][9]
//   aplus/-  [e][face][p][9]     nb, jh  [e][4]
// One CTA handles kTE elements; shared-memory work arrays are [row][p][kTE].  Every
// global-matrix product runs with one thread per (output row, element, group of 9 quantity
// columns): a CSR entry (value, column) is loaded once and applied to the 9 columns held in
// registers, so the products cost about one shared-memory load per FMA.
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

template <int P>
__device__ __forceinline__ int idx3(int k, int p, int e) { return (k * P + p) * kTE + e; }

// acc[p] += sum over CSR row `row` of M: val * W[col][p][e], p < PO (W has PW quantities)
template <int PO, int PW>
__device__ __forceinline__ void csr_row(const Csr& M, int row, const double* W, int e, double (&acc)[PO]) {
  const int t1 = M.ptr[row + 1];
  for (int t = M.ptr[row]; t < t1; ++t) {
    const double v = M.val[t];
    const double* w = W + idx3<PW>(M.col[t], 0, e);
#pragma unroll
    for (int p = 0; p < PO; ++p) acc[p] = fma(v, w[p * kTE], acc[p]);
  }
}

// X^c[l][p][e] = sum_j A*^c[p][scol_j] D[l][scol_j][e], one thread per (row l, element e)
// (the D loads are shared by the three c); star coefficients from shared memory.
template <int P>
__device__ __forceinline__ void make_x(const double* D, const double* ST, double* X, int B) {
  const int SZ = B * P * kTE;
  for (int i = threadIdx.x; i < B * kTE; i += blockDim.x) {  // (row l, element e), all c and p
    const int e = i % kTE, l = i / kTE;
    const double* d = D + idx3<P>(l, 0, e);
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const double* a = ST + ((e * 3 + c) * P + p) * 3;
        double s = a[0] * d[c_scols[p][0] * kTE];
        s = fma(a[1], d[c_scols[p][1] * kTE], s);
        s = fma(a[2], d[c_scols[p][2] * kTE], s);
        X[c * SZ + idx3<P>(l, p, e)] = s;
      }
  }
}

// Shared-memory copy of a CSR matrix (values, then columns, then row pointers).
__device__ __forceinline__ Csr stage_csr(const Csr& g, int rows, int nnz, double* dst) {
  double* val = dst;
  int* col = reinterpret_cast<int*>(val + nnz);
  int* ptr = col + nnz;
  for (int i = threadIdx.x; i < nnz; i += blockDim.x) {
    val[i] = g.val[i];
    col[i] = g.col[i];
  }
  for (int i = threadIdx.x; i <= rows; i += blockDim.x) ptr[i] = g.ptr[i];
  return Csr{ptr, col, val};
}
__host__ __device__ __forceinline__ int csr_doubles(int rows, int nnz) { return nnz + (nnz + rows + 2) / 2 + 1; }

// Persistent over groups of kTE elements; KSM: the CK and volume CSR matrices staged in
// shared memory once per CTA (when they fit).
template <int P, bool KSM>
__global__ void __launch_bounds__(256) gen_local(const GenParams prm) {
  constexpr int kG = P / 9;  // groups of 9 quantity columns per (row, element): one thread each
  extern __shared__ double sm[];
  const int B = prm.B, Bt = prm.Bt;
  const int SZ = B * P * kTE;
  const int XS = 3 * SZ > 4 * Bt * (9 + P) * kTE ? 3 * SZ : 4 * Bt * (9 + P) * kTE;
  double* const base = sm;
  double* ST = base + 3 * SZ + XS;     // [kTE][3][P][3] star coefficients
  double* SRC = ST + kTE * 3 * P * 3;  // [kTE][P][9] source coefficients (P = 27)
  Csr Kt{prm.kt_ptr, prm.kt_col, prm.kt_val}, Kh{prm.kh_ptr, prm.kh_col, prm.kh_val};
  if (KSM) {
    double* c0 = SRC + kTE * P * 9;
    Kt = stage_csr(Kt, 3 * B, prm.kt_nnz, c0);
    Kh = stage_csr(Kh, 3 * B, prm.kh_nnz, c0 + csr_doubles(3 * B, prm.kt_nnz));
  }
  const Csr Rt{prm.rt_ptr, prm.rt_col, prm.rt_val}, R{prm.r_ptr, prm.r_col, prm.r_val};
  const int64_t nblk = (prm.n + kTE - 1) / kTE;
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
  double* D = base;
  double* Dn = D + SZ;
  double* I = Dn + SZ;
  double* X = I + SZ;                  // [3][B][P][kTE]; later: traces / flux staging
  const int64_t e0 = prm.e0 + blk * kTE;
  const int64_t left = prm.e0 + prm.n - e0;
  const int ne = static_cast<int>(left < kTE ? left : kTE);
  __syncthreads();  // previous group done with the shared regions
  // load Q, I = dt Q, coefficients
  for (int i = threadIdx.x; i < SZ; i += blockDim.x) {
    const int e = i % kTE, kp = i / kTE, p = kp % P, k = kp / P;
    const double q = e < ne ? prm.Q[((e0 + e) * P + p) * B + k] : 0.0;
    D[i] = q;
    I[i] = prm.dt * q;
  }
  for (int i = threadIdx.x; i < kTE * 3 * P * 3; i += blockDim.x) {
    const int e = i / (3 * P * 3);
    ST[i] = e < ne ? prm.star[(e0 + e) * 3 * P * 3 + i % (3 * P * 3)] : 0.0;
  }
  if (P == 27)
    for (int i = threadIdx.x; i < kTE * P * 9; i += blockDim.x) {
      const int e = i / (P * 9);
      SRC[i] = (prm.src && e < ne) ? prm.src[(e0 + e) * P * 9 + i % (P * 9)] : 0.0;
    }
  __syncthreads();
  // CK recursion (scaled derivatives, reading R12) and time integral
  for (int d = 0; d < prm.N; ++d) {
    make_x<P>(D, ST, X, B);
    __syncthreads();
    const double sc = prm.scal[d], ic = prm.scal[prm.N + d];
    for (int i = threadIdx.x; i < B * kTE * kG; i += blockDim.x) {  // (row k, group g, element e)
      const int e = i % kTE, g = (i / kTE) % kG, k = i / (kTE * kG);
      double s[9];
#pragma unroll
      for (int p = 0; p < 9; ++p) s[p] = 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) csr_row<9, P>(Kt, c * B + k, X + c * SZ + 9 * g * kTE, e, s);
      if (P == 27) {
        const double* dk = D + idx3<P>(k, 0, e);
#pragma unroll
        for (int q = 0; q < 9; ++q) {
          const int p = 9 * g + q;
#pragma unroll
          for (int j = 0; j < 9; ++j) s[q] = fma(SRC[(e * P + p) * 9 + j], dk[c_ecols[p][j] * kTE], s[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        const int p = 9 * g + q;
        const double v = sc * s[q];
        Dn[idx3<P>(k, p, e)] = v;
        I[idx3<P>(k, p, e)] = fma(ic, v, I[idx3<P>(k, p, e)]);
      }
    }
    __syncthreads();
    double* t = D;
    D = Dn;
    Dn = t;
  }
  // volume: U = sum_c Khat^c (I A*^cT) + I E^T
  make_x<P>(I, ST, X, B);
  __syncthreads();
  double* U = Dn;  // accumulated update [B][P][kTE]
  for (int i = threadIdx.x; i < B * kTE * kG; i += blockDim.x) {
    const int e = i % kTE, g = (i / kTE) % kG, k = i / (kTE * kG);
    double s[9];
#pragma unroll
    for (int p = 0; p < 9; ++p) s[p] = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) csr_row<9, P>(Kh, c * B + k, X + c * SZ + 9 * g * kTE, e, s);
    if (P == 27) {
      const double* ik = I + idx3<P>(k, 0, e);
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        const int p = 9 * g + q;
#pragma unroll
        for (int j = 0; j < 9; ++j) s[q] = fma(SRC[(e * P + p) * 9 + j], ik[c_ecols[p][j] * kTE], s[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) U[idx3<P>(k, 9 * g + q, e)] = s[q];
  }
  __syncthreads();
  // traces T_i[m][q] = sum_l R^i[l][m] I[l][q], q < 9  -> X region [4][Bt][9][kTE] and global
  const int TS = Bt * 9 * kTE;
  for (int i = threadIdx.x; i < 4 * Bt * kTE; i += blockDim.x) {
    const int e = i % kTE, fm = i / kTE, m = fm % Bt, f = fm / Bt;
    double s[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) s[q] = 0.0;
    csr_row<9, P>(Rt, f * Bt + m, I, e, s);
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      X[f * TS + (m * 9 + q) * kTE + e] = s[q];
      if (e < ne) prm.traces[(((e0 + e) * 4 + f) * Bt + m) * 9 + q] = s[q];
    }
  }
  __syncthreads();
  // local flux: Y_i[m][p] = sum_j A+_i[p][j] T_i[m][j]  -> X + 4 TS region [4][Bt][P][kTE];
  // thread (face, p, e) holds its 9 solver coefficients
  double* Y = X + 4 * TS;
  const int YS = Bt * P * kTE;
  for (int i = threadIdx.x; i < 4 * P * kTE; i += blockDim.x) {
    const int e = i % kTE, fp = i / kTE, p = fp % P, f = fp / P;
    double a[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) a[j] = e < ne ? prm.aplus[(((e0 + e) * 4 + f) * P + p) * 9 + j] : 0.0;
    for (int m = 0; m < Bt; ++m) {
      const double* t = X + f * TS + m * 9 * kTE + e;
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < 9; ++j) s = fma(a[j], t[j * kTE], s);
      Y[f * YS + (m * P + p) * kTE + e] = s;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < B * kTE * kG; i += blockDim.x) {
    const int e = i % kTE, g = (i / kTE) % kG, k = i / (kTE * kG);
    double s[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) s[q] = U[idx3<P>(k, 9 * g + q, e)];
#pragma unroll
    for (int f = 0; f < 4; ++f) csr_row<9, P>(R, f * B + k, Y + f * YS + 9 * g * kTE, e, s);
    if (e < ne)
#pragma unroll
      for (int q = 0; q < 9; ++q) prm.Q[((e0 + e) * P + 9 * g + q) * B + k] += s[q];
  }
  }  // element groups
}

template <int P>
__global__ void __launch_bounds__(256) gen_neigh(const GenParams prm) {
  constexpr int kG = P / 9;
  extern __shared__ double sm[];
  const int B = prm.B, Bt = prm.Bt;
  const int64_t e0 = prm.e0 + static_cast<int64_t>(blockIdx.x) * kTE;
  const int64_t left = prm.e0 + prm.n - e0;
  const int ne = static_cast<int>(left < kTE ? left : kTE);
  const Csr R{prm.r_ptr, prm.r_col, prm.r_val}, Fh{prm.f_ptr, prm.f_col, prm.f_val};
  const int TS = Bt * 9 * kTE, YS = Bt * P * kTE;
  double* Z = sm;            // [4][Bt][9][kTE]
  double* Y = Z + 4 * TS;    // [4][Bt][P][kTE]
  // rotated neighbour traces z = f^h t: thread (face, m, e), all 9 quantities
  for (int i = threadIdx.x; i < 4 * Bt * kTE; i += blockDim.x) {
    const int e = i % kTE, fm = i / kTE, m = fm % Bt, f = fm / Bt;
    double s[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) s[q] = 0.0;
    if (e < ne) {
      const int64_t nbe = prm.nb[(e0 + e) * 4 + f];
      const int jh = prm.jh[(e0 + e) * 4 + f];
      const int j = jh & 3, h = jh >> 2;
      const double* src = prm.traces + ((nbe * 4 + j) * Bt) * 9;
      const int row = h * Bt + m;
      for (int t = Fh.ptr[row]; t < Fh.ptr[row + 1]; ++t) {
        const double v = Fh.val[t];
        const double* sr = src + Fh.col[t] * 9;
#pragma unroll
        for (int q = 0; q < 9; ++q) s[q] = fma(v, sr[q], s[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) Z[f * TS + (m * 9 + q) * kTE + e] = s[q];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4 * P * kTE; i += blockDim.x) {
    const int e = i % kTE, fp = i / kTE, p = fp % P, f = fp / P;
    double a[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) a[j] = e < ne ? prm.aminus[(((e0 + e) * 4 + f) * P + p) * 9 + j] : 0.0;
    for (int m = 0; m < Bt; ++m) {
      const double* z = Z + f * TS + m * 9 * kTE + e;
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < 9; ++j) s = fma(a[j], z[j * kTE], s);
      Y[f * YS + (m * P + p) * kTE + e] = s;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < B * kTE * kG; i += blockDim.x) {
    const int e = i % kTE, g = (i / kTE) % kG, k = i / (kTE * kG);
    double s[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) s[q] = 0.0;
#pragma unroll
    for (int f = 0; f < 4; ++f) csr_row<9, P>(R, f * B + k, Y + f * YS + 9 * g * kTE, e, s);
    if (e < ne)
#pragma unroll
      for (int q = 0; q < 9; ++q) prm.Q[((e0 + e) * P + 9 * g + q) * B + k] += s[q];
  }
}

}  // namespace gen

size_t gen_local_smem(int B, int Bt, int P) {
  const size_t SZ = static_cast<size_t>(B) * P * gen::kTE;
  const size_t extra = static_cast<size_t>(4) * Bt * 9 * gen::kTE + static_cast<size_t>(4) * Bt * P * gen::kTE;
  const size_t coef = static_cast<size_t>(gen::kTE) * (3 * P * 3 + P * 9);
  return (3 * SZ + (3 * SZ > extra ? 3 * SZ : extra) + coef) * sizeof(double);
}
static size_t gen_local_smem_ksm(const GenParams& p) {
  return gen_local_smem(p.B, p.Bt, p.P) +
         (gen::csr_doubles(3 * p.B, p.kt_nnz) + gen::csr_doubles(3 * p.B, p.kh_nnz)) * sizeof(double);
}
static bool gen_ksm(const GenParams& p) { return gen_local_smem_ksm(p) <= 227 * 1024; }
size_t gen_neigh_smem(int Bt, int P) {
  return (static_cast<size_t>(4) * Bt * 9 * gen::kTE + static_cast<size_t>(4) * Bt * P * gen::kTE) * sizeof(double);
}

cudaError_t gen_configure(int B, int Bt, int P, const int (*ecols)[9], const int (*scols)[3]) {
  cudaError_t e = cudaMemcpyToSymbol(gen::c_ecols, ecols, sizeof(int) * 27 * 9);
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(gen::c_scols, scols, sizeof(int) * 27 * 3);
  const void* fls[4] = {reinterpret_cast<const void*>(&gen::gen_local<9, false>),
                        reinterpret_cast<const void*>(&gen::gen_local<9, true>),
                        reinterpret_cast<const void*>(&gen::gen_local<27, false>),
                        reinterpret_cast<const void*>(&gen::gen_local<27, true>)};
  const void* fn = P == 27 ? reinterpret_cast<const void*>(&gen::gen_neigh<27>) : reinterpret_cast<const void*>(&gen::gen_neigh<9>);
  for (int i = (P == 27 ? 2 : 0); e == cudaSuccess && i < (P == 27 ? 4 : 2); ++i)
    e = cudaFuncSetAttribute(fls[i], cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(gen_neigh_smem(Bt, P)));
  return e;
}

cudaError_t gen_launch(const GenParams& p, bool local, cudaStream_t s) {
  const int64_t blocks = (p.n + gen::kTE - 1) / gen::kTE;
  if (blocks <= 0) return cudaSuccess;
  const unsigned nb = static_cast<unsigned>(blocks);
  if (local) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const unsigned g = static_cast<unsigned>(blocks < sms ? blocks : sms);  // persistent
    const bool ksm = gen_ksm(p);
    const size_t smem = ksm ? gen_local_smem_ksm(p) : gen_local_smem(p.B, p.Bt, p.P);
    if (p.P == 27) {
      if (ksm) gen::gen_local<27, true><<<g, 256, smem, s>>>(p);
      else gen::gen_local<27, false><<<g, 256, smem, s>>>(p);
    } else {
      if (ksm) gen::gen_local<9, true><<<g, 256, smem, s>>>(p);
      else gen::gen_local<9, false><<<g, 256, smem, s>>>(p);
    }
  } else {
    if (p.P == 27) gen::gen_neigh<27><<<nb, 256, gen_neigh_smem(p.Bt, p.P), s>>>(p);
    else gen::gen_neigh<9><<<nb, 256, gen_neigh_smem(p.Bt, p.P), s>>>(p);
  }
  return cudaGetLastError();
}

int gen_tile_elems() { return gen::kTE; }

}  // namespace ydg
