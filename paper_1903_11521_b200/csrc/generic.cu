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

constexpr int kTE = 4;  // elements per CTA (default; the local kernel takes 2 where 4 does not fit)

// Column patterns, one table per quantity count (a P = 9 and a P = 27 handle may coexist in
// a process): star matrices (3 columns per row), viscoelastic source (9 per row).
__constant__ int c_scols9[9][3];
__constant__ int c_scols27[27][3];
__constant__ int c_ecols27[27][9];
template <int P>
__device__ __forceinline__ int scol(int p, int j) { return P == 27 ? c_scols27[p][j] : c_scols9[p][j]; }

struct Csr {
  const int* ptr;
  const int* col;
  const double* val;
};

template <int P, int TE>
__device__ __forceinline__ int idx3(int k, int p, int e) { return (k * P + p) * TE + e; }

// acc[p] += sum over CSR row `row` of M: val * W[col][p][e], p < PO (W has PW quantities)
template <int PO, int PW, int TE>
__device__ __forceinline__ void csr_row(const Csr& M, int row, const double* W, int e, double (&acc)[PO]) {
  const int t1 = M.ptr[row + 1];
  for (int t = M.ptr[row]; t < t1; ++t) {
    const double v = M.val[t];
    const double* w = W + idx3<PW, TE>(M.col[t], 0, e);
#pragma unroll
    for (int p = 0; p < PO; ++p) acc[p] = fma(v, w[p * TE], acc[p]);
  }
}

// X^c[l][p][e] = sum_j A*^c[p][scol_j] D[l][scol_j][e], one thread per (row l, element e)
// (the D loads are shared by the three c); star coefficients from shared memory.
template <int P, int TE>
__device__ __forceinline__ void make_x(const double* D, const double* ST, double* X, int B) {
  const int SZ = B * P * TE;
  for (int i = threadIdx.x; i < B * TE; i += blockDim.x) {  // (row l, element e), all c and p
    const int e = i % TE, l = i / TE;
    const double* d = D + idx3<P, TE>(l, 0, e);
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const double* a = ST + ((e * 3 + c) * P + p) * 3;
        double s = a[0] * d[scol<P>(p, 0) * TE];
        s = fma(a[1], d[scol<P>(p, 1) * TE], s);
        s = fma(a[2], d[scol<P>(p, 2) * TE], s);
        X[c * SZ + idx3<P, TE>(l, p, e)] = s;
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

// Persistent over groups of TE elements; KSM: the CK and volume CSR matrices staged in
// shared memory once per CTA (when they fit).
template <int P, bool KSM, int TE>
__global__ void __launch_bounds__(256) gen_local(const GenParams prm) {
  constexpr int kG = P / 9;  // groups of 9 quantity columns per (row, element): one thread each
  extern __shared__ double sm[];
  const int B = prm.B, Bt = prm.Bt;
  const int SZ = B * P * TE;
  const int XS = 3 * SZ > 4 * Bt * (9 + P) * TE ? 3 * SZ : 4 * Bt * (9 + P) * TE;
  double* const base = sm;
  double* ST = base + 3 * SZ + XS;     // [TE][3][P][3] star coefficients
  double* SRC = ST + TE * 3 * P * 3;  // [TE][P][9] source coefficients (P = 27)
  Csr Kt{prm.kt_ptr, prm.kt_col, prm.kt_val}, Kh{prm.kh_ptr, prm.kh_col, prm.kh_val};
  if (KSM) {
    double* c0 = SRC + TE * P * 9;
    Kt = stage_csr(Kt, 3 * B, prm.kt_nnz, c0);
    Kh = stage_csr(Kh, 3 * B, prm.kh_nnz, c0 + csr_doubles(3 * B, prm.kt_nnz));
  }
  const Csr Rt{prm.rt_ptr, prm.rt_col, prm.rt_val}, R{prm.r_ptr, prm.r_col, prm.r_val};
  const int64_t nblk = (prm.n + TE - 1) / TE;
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
  double* D = base;
  double* Dn = D + SZ;
  double* I = Dn + SZ;
  double* X = I + SZ;                  // [3][B][P][TE]; later: traces / flux staging
  const int64_t e0 = prm.e0 + blk * TE;
  const int64_t left = prm.e0 + prm.n - e0;
  const int ne = static_cast<int>(left < TE ? left : TE);
  __syncthreads();  // previous group done with the shared regions
  // load Q, I = dt Q, coefficients
  for (int i = threadIdx.x; i < SZ; i += blockDim.x) {
    const int e = i % TE, kp = i / TE, p = kp % P, k = kp / P;
    const double q = e < ne ? prm.Q[((e0 + e) * P + p) * B + k] : 0.0;
    D[i] = q;
    I[i] = prm.dt * q;
  }
  for (int i = threadIdx.x; i < TE * 3 * P * 3; i += blockDim.x) {
    const int e = i / (3 * P * 3);
    ST[i] = e < ne ? prm.star[(e0 + e) * 3 * P * 3 + i % (3 * P * 3)] : 0.0;
  }
  if (P == 27)
    for (int i = threadIdx.x; i < TE * P * 9; i += blockDim.x) {
      const int e = i / (P * 9);
      SRC[i] = (prm.src && e < ne) ? prm.src[(e0 + e) * P * 9 + i % (P * 9)] : 0.0;
    }
  __syncthreads();
  // CK recursion (scaled derivatives, reading R12) and time integral
  for (int d = 0; d < prm.N; ++d) {
    make_x<P, TE>(D, ST, X, B);
    __syncthreads();
    const double sc = prm.scal[d], ic = prm.scal[prm.N + d];
    for (int i = threadIdx.x; i < B * TE * kG; i += blockDim.x) {  // (row k, group g, element e)
      const int e = i % TE, g = (i / TE) % kG, k = i / (TE * kG);
      double s[9];
#pragma unroll
      for (int p = 0; p < 9; ++p) s[p] = 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) csr_row<9, P, TE>(Kt, c * B + k, X + c * SZ + 9 * g * TE, e, s);
      if (P == 27) {
        const double* dk = D + idx3<P, TE>(k, 0, e);
#pragma unroll
        for (int q = 0; q < 9; ++q) {
          const int p = 9 * g + q;
#pragma unroll
          for (int j = 0; j < 9; ++j) s[q] = fma(SRC[(e * P + p) * 9 + j], dk[c_ecols27[p][j] * TE], s[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        const int p = 9 * g + q;
        const double v = sc * s[q];
        Dn[idx3<P, TE>(k, p, e)] = v;
        I[idx3<P, TE>(k, p, e)] = fma(ic, v, I[idx3<P, TE>(k, p, e)]);
      }
    }
    __syncthreads();
    double* t = D;
    D = Dn;
    Dn = t;
  }
  // volume: U = sum_c Khat^c (I A*^cT) + I E^T
  make_x<P, TE>(I, ST, X, B);
  __syncthreads();
  double* U = Dn;  // accumulated update [B][P][TE]
  for (int i = threadIdx.x; i < B * TE * kG; i += blockDim.x) {
    const int e = i % TE, g = (i / TE) % kG, k = i / (TE * kG);
    double s[9];
#pragma unroll
    for (int p = 0; p < 9; ++p) s[p] = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) csr_row<9, P, TE>(Kh, c * B + k, X + c * SZ + 9 * g * TE, e, s);
    if (P == 27) {
      const double* ik = I + idx3<P, TE>(k, 0, e);
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        const int p = 9 * g + q;
#pragma unroll
        for (int j = 0; j < 9; ++j) s[q] = fma(SRC[(e * P + p) * 9 + j], ik[c_ecols27[p][j] * TE], s[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) U[idx3<P, TE>(k, 9 * g + q, e)] = s[q];
  }
  __syncthreads();
  // traces T_i[m][q] = sum_l R^i[l][m] I[l][q], q < 9  -> X region [4][Bt][9][TE] and global
  const int TS = Bt * 9 * TE;
  for (int i = threadIdx.x; i < 4 * Bt * TE; i += blockDim.x) {
    const int e = i % TE, fm = i / TE, m = fm % Bt, f = fm / Bt;
    double s[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) s[q] = 0.0;
    csr_row<9, P, TE>(Rt, f * Bt + m, I, e, s);
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      X[f * TS + (m * 9 + q) * TE + e] = s[q];
      if (e < ne) prm.traces[(((e0 + e) * 4 + f) * Bt + m) * 9 + q] = s[q];
    }
  }
  __syncthreads();
  // local flux: Y_i[m][p] = sum_j A+_i[p][j] T_i[m][j]  -> X + 4 TS region [4][Bt][P][TE];
  // thread (face, p, e) holds its 9 solver coefficients
  double* Y = X + 4 * TS;
  const int YS = Bt * P * TE;
  for (int i = threadIdx.x; i < 4 * P * TE; i += blockDim.x) {
    const int e = i % TE, fp = i / TE, p = fp % P, f = fp / P;
    double a[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) a[j] = e < ne ? prm.aplus[(((e0 + e) * 4 + f) * P + p) * 9 + j] : 0.0;
    for (int m = 0; m < Bt; ++m) {
      const double* t = X + f * TS + m * 9 * TE + e;
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < 9; ++j) s = fma(a[j], t[j * TE], s);
      Y[f * YS + (m * P + p) * TE + e] = s;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < B * TE * kG; i += blockDim.x) {
    const int e = i % TE, g = (i / TE) % kG, k = i / (TE * kG);
    double s[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) s[q] = U[idx3<P, TE>(k, 9 * g + q, e)];
#pragma unroll
    for (int f = 0; f < 4; ++f) csr_row<9, P, TE>(R, f * B + k, Y + f * YS + 9 * g * TE, e, s);
    if (e < ne)
#pragma unroll
      for (int q = 0; q < 9; ++q) prm.Q[((e0 + e) * P + 9 * g + q) * B + k] += s[q];
  }
  }  // element groups
}

template <int P, int TE>
__global__ void __launch_bounds__(256) gen_neigh(const GenParams prm) {
  constexpr int kG = P / 9;
  extern __shared__ double sm[];
  const int B = prm.B, Bt = prm.Bt;
  const int64_t e0 = prm.e0 + static_cast<int64_t>(blockIdx.x) * TE;
  const int64_t left = prm.e0 + prm.n - e0;
  const int ne = static_cast<int>(left < TE ? left : TE);
  const Csr R{prm.r_ptr, prm.r_col, prm.r_val}, Fh{prm.f_ptr, prm.f_col, prm.f_val};
  const int TS = Bt * 9 * TE, YS = Bt * P * TE;
  double* Z = sm;            // [4][Bt][9][TE]
  double* Y = Z + 4 * TS;    // [4][Bt][P][TE]
  // rotated neighbour traces z = f^h t: thread (face, m, e), all 9 quantities
  for (int i = threadIdx.x; i < 4 * Bt * TE; i += blockDim.x) {
    const int e = i % TE, fm = i / TE, m = fm % Bt, f = fm / Bt;
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
    for (int q = 0; q < 9; ++q) Z[f * TS + (m * 9 + q) * TE + e] = s[q];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4 * P * TE; i += blockDim.x) {
    const int e = i % TE, fp = i / TE, p = fp % P, f = fp / P;
    double a[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) a[j] = e < ne ? prm.aminus[(((e0 + e) * 4 + f) * P + p) * 9 + j] : 0.0;
    for (int m = 0; m < Bt; ++m) {
      const double* z = Z + f * TS + m * 9 * TE + e;
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < 9; ++j) s = fma(a[j], z[j * TE], s);
      Y[f * YS + (m * P + p) * TE + e] = s;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < B * TE * kG; i += blockDim.x) {
    const int e = i % TE, g = (i / TE) % kG, k = i / (TE * kG);
    double s[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) s[q] = 0.0;
#pragma unroll
    for (int f = 0; f < 4; ++f) csr_row<9, P, TE>(R, f * B + k, Y + f * YS + 9 * g * TE, e, s);
    if (e < ne)
#pragma unroll
      for (int q = 0; q < 9; ++q) prm.Q[((e0 + e) * P + 9 * g + q) * B + k] += s[q];
  }
}

}  // namespace gen

static constexpr size_t kSmemMax = 227 * 1024;
size_t gen_local_smem(int B, int Bt, int P, int te) {
  const size_t SZ = static_cast<size_t>(B) * P * te;
  const size_t extra = static_cast<size_t>(4) * Bt * 9 * te + static_cast<size_t>(4) * Bt * P * te;
  const size_t coef = static_cast<size_t>(te) * (3 * P * 3 + P * 9);
  return (3 * SZ + (3 * SZ > extra ? 3 * SZ : extra) + coef) * sizeof(double);
}
// elements per CTA of the local kernel: 4, or 2 where 4 does not fit (P = 27 at N >= 5);
// 0 if neither fits (ydg_create then reports YDG_ERR_UNSUPPORTED)
int gen_local_te(int B, int Bt, int P) {
  if (gen_local_smem(B, Bt, P, 4) <= kSmemMax) return 4;
  if (gen_local_smem(B, Bt, P, 2) <= kSmemMax) return 2;
  return 0;
}
static size_t gen_local_smem_ksm(const GenParams& p, int te) {
  return gen_local_smem(p.B, p.Bt, p.P, te) +
         (gen::csr_doubles(3 * p.B, p.kt_nnz) + gen::csr_doubles(3 * p.B, p.kh_nnz)) * sizeof(double);
}
size_t gen_neigh_smem(int Bt, int P) {
  return (static_cast<size_t>(4) * Bt * 9 * gen::kTE + static_cast<size_t>(4) * Bt * P * gen::kTE) * sizeof(double);
}

cudaError_t gen_configure(int B, int Bt, int P, const int (*ecols)[9], const int (*scols)[3]) {
  if (gen_local_te(B, Bt, P) == 0 || gen_neigh_smem(Bt, P) > kSmemMax) return cudaErrorInvalidConfiguration;
  // the patterns are fixed functions of P; each P has its own tables
  cudaError_t e = P == 27 ? cudaMemcpyToSymbol(gen::c_scols27, scols, sizeof(int) * 27 * 3)
                          : cudaMemcpyToSymbol(gen::c_scols9, scols, sizeof(int) * 9 * 3);
  if (e == cudaSuccess && P == 27) e = cudaMemcpyToSymbol(gen::c_ecols27, ecols, sizeof(int) * 27 * 9);
  const void* fls[] = {reinterpret_cast<const void*>(&gen::gen_local<9, false, 4>),
                       reinterpret_cast<const void*>(&gen::gen_local<9, true, 4>),
                       reinterpret_cast<const void*>(&gen::gen_local<9, false, 2>),
                       reinterpret_cast<const void*>(&gen::gen_local<9, true, 2>),
                       reinterpret_cast<const void*>(&gen::gen_local<27, false, 4>),
                       reinterpret_cast<const void*>(&gen::gen_local<27, true, 4>),
                       reinterpret_cast<const void*>(&gen::gen_local<27, false, 2>),
                       reinterpret_cast<const void*>(&gen::gen_local<27, true, 2>)};
  const void* fn = P == 27 ? reinterpret_cast<const void*>(&gen::gen_neigh<27, gen::kTE>)
                           : reinterpret_cast<const void*>(&gen::gen_neigh<9, gen::kTE>);
  for (int i = (P == 27 ? 4 : 0); e == cudaSuccess && i < (P == 27 ? 8 : 4); ++i)
    e = cudaFuncSetAttribute(fls[i], cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemMax));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(gen_neigh_smem(Bt, P)));
  return e;
}

template <int P, int TE>
static void launch_local(const GenParams& p, cudaStream_t s, int sms) {
  const int64_t blocks = (p.n + TE - 1) / TE;
  const unsigned g = static_cast<unsigned>(blocks < sms ? blocks : sms);  // persistent
  const size_t ksm_bytes = gen_local_smem_ksm(p, TE);
  if (ksm_bytes <= kSmemMax) gen::gen_local<P, true, TE><<<g, 256, ksm_bytes, s>>>(p);
  else gen::gen_local<P, false, TE><<<g, 256, gen_local_smem(p.B, p.Bt, p.P, TE), s>>>(p);
}

cudaError_t gen_launch(const GenParams& p, bool local, cudaStream_t s) {
  if (p.n <= 0) return cudaSuccess;
  if (local) {
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int te = gen_local_te(p.B, p.Bt, p.P);
    if (te == 0) return cudaErrorInvalidConfiguration;
    if (p.P == 27) {
      if (te == 4) launch_local<27, 4>(p, s, sms);
      else launch_local<27, 2>(p, s, sms);
    } else {
      if (te == 4) launch_local<9, 4>(p, s, sms);
      else launch_local<9, 2>(p, s, sms);
    }
  } else {
    const unsigned nb = static_cast<unsigned>((p.n + gen::kTE - 1) / gen::kTE);
    if (p.P == 27) gen::gen_neigh<27, gen::kTE><<<nb, 256, gen_neigh_smem(p.Bt, p.P), s>>>(p);
    else gen::gen_neigh<9, gen::kTE><<<nb, 256, gen_neigh_smem(p.Bt, p.P), s>>>(p);
  }
  return cudaGetLastError();
}

int gen_tile_elems() { return gen::kTE; }

}  // namespace ydg
