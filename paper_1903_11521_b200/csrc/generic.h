// Generic (any N, any P, fp64) ADER-DG kernels: see generic.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace ydg {

struct GenParams {
  double* Q;            // [e][p][k]
  double* traces;       // [e][face][m][9]
  const double* star;   // [e][c][p][3]
  const double* src;    // [e][p][9] or null (elastic)
  const double* aplus;  // [e][face][p][9]
  const double* aminus;
  const int64_t* nb;    // [e][4]
  const int8_t* jh;     // [e][4]  j | h << 2
  const int *kt_ptr, *kt_col, *kh_ptr, *kh_col, *rt_ptr, *rt_col, *r_ptr, *r_col, *f_ptr, *f_col;
  const double *kt_val, *kh_val, *rt_val, *r_val, *f_val;
  int kt_nnz, kh_nnz;   // nonzeros of the CK / volume CSR matrices (staged in shared memory)
  int N, B, Bt, P;
  int64_t e0, n;        // element range of this launch
  double dt;
  double scal[12];      // dt/(d+1), d < N; dt/(d+2), d < N
  double wratio[3];     // omega_l / omega_0: the memory-variable star rows of mechanism l are
                        // wratio[l] x those of mechanism 0 (checked at upload; visco.cu)
};

size_t gen_local_smem(int B, int Bt, int P, int te);
int gen_local_te(int B, int Bt, int P);
size_t gen_neigh_smem(int Bt, int P);
cudaError_t gen_configure(int B, int Bt, int P, const int (*ecols)[9], const int (*scols)[3]);
cudaError_t gen_launch(const GenParams& p, bool local, cudaStream_t s);
int gen_tile_elems();

// Viscoelastic (P = 27) local and neighbour-flux kernels on FP64 tensor cores, orders 1..4
// (visco.cu).
bool visco_supported(int N, int P);
cudaError_t visco_configure(int N, const int (*scols)[3]);
cudaError_t visco_launch_local(const GenParams& p, cudaStream_t s);
cudaError_t visco_launch_neigh(const GenParams& p, cudaStream_t s);

}  // namespace ydg
