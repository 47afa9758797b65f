// CUDA kernels of the ADER-DG element update (sm_100a).  Internal header.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ydg {

constexpr int kLanes = 32;   // elements per tile of the fp32 kernels
// fp64 tensor-core kernels: elements per tile (8 or 16), warps per work group (3 per 8
// elements), groups per SM (12 warps per SM: three per sub-partition).  Measured (c1): 8-element
// tiles in four 3-warp groups per CTA 14.69 / 7.60 ms (local / flux) vs 16-element tiles in two
// 6-warp groups 14.82 / 7.88 ms
#ifndef YDG_DM_LANES
#define YDG_DM_LANES 8
#endif
constexpr int kDmLanes = YDG_DM_LANES;
constexpr int kDmWarps = 3 * (kDmLanes / 8);
constexpr int kDmCtasPerSm = 12 / kDmWarps;
// fp64 flux kernel: 3-warp groups (8-element halves) per CTA.  1: one group per CTA, four
// CTAs per SM; 4: one CTA per SM whose four groups share the lift's A fragments staged in
// shared memory (named barriers per group).
// fp64 local kernel: 1: kDmCtasPerSm CTAs per SM; > 1: one CTA per SM of that many work groups
// (kDmCtasPerSm of them: four 3-warp groups at 8-element tiles, two 6-warp groups at 16)
// sharing CK step 0's and (part of) the volume's A fragments in shared memory
#ifndef YDG_LOCAL_GROUPS
#define YDG_LOCAL_GROUPS (YDG_DM_LANES == 8 ? 4 : 2)
#endif
constexpr int kLocalGroups = YDG_LOCAL_GROUPS;
#ifndef YDG_FLUX_GROUPS
#define YDG_FLUX_GROUPS 4
#endif
constexpr int kFluxGroups = YDG_FLUX_GROUPS;
constexpr int kMaxN = 6;

template <typename T>
struct StepParams {
  T* Q;                  // [tile][k][p][L]  DOFs (updated in place); L = 32 (fp32), 16 (fp64)
  T* traces;             // time-integrated face traces R^iT I: fp32 [tile][face][m][q][32],
                         // fp64 [tile][face][lane][TS] (element-face blocks [m][q])
  const T* star;         // [tile][c][p][3][32]
  const T* aplus;        // fp32: [tile][face][p][q][32] (-2|S|/detJ folded in);
                         // fp64: factored flux solvers [tile][face][kFaceCoeffs][32]
  const T* aminus;       // fp32: [tile][face][p][q][32]; fp64: unused
  const int32_t* nb;     // [tile][face][32] neighbour element (local index incl. ghosts)
  const int8_t* jh;      // [tile][face][max(L, 16)] j | (h << 2)
  int64_t tile0;         // first tile handled by this launch
  int64_t ntiles;        // number of tiles handled
  T scal[2 * kMaxN];     // dt/(d+1), d < N ; dt/(d+2), d < N
  T dt;
  int tr_only;           // fp64 local kernel: traces of I only, no volume update (LTS)
  const T* traces_in;    // fp64 fused kernel: the previous step's traces (its flux phase's input)
};

// host launchers (kernels.cu)
template <typename T>
cudaError_t launch_local(int N, const StepParams<T>& p, int grid, cudaStream_t s);
template <typename T>
cudaError_t launch_neigh(int N, const StepParams<T>& p, int grid, cudaStream_t s);
// fp64 fused step kernel (flux of the previous step + local part of this one, per tile)
cudaError_t launch_fused(int N, const StepParams<double>& p, int grid, cudaStream_t s);
size_t fused_smem_bytes(int N);
template <typename T>
cudaError_t launch_to_tiled(int P, int B, int L, const T* canon, T* tiled, int64_t first, int64_t count,
                            const int32_t* slot_of, cudaStream_t s);
template <typename T>
cudaError_t launch_to_canonical(int P, int B, int L, const T* tiled, T* canon, int64_t first,
                                int64_t count, const int32_t* slot_of, cudaStream_t s);
// LTS: per entry (dst, a, b) element slots, all four faces: mode 0 dst = a, 1 dst = a - b,
// 2 dst += a (fp64 trace layout [tile][face][lane][TS])
cudaError_t launch_trace_combine(double* traces, const int64_t* lst, int64_t n, int TS, int L, int mode,
                                 cudaStream_t s);
// max |Q| over owned elements; L > 0: tiled [tile][k][p][L], L = 0: canonical [e][p][k]
template <typename T>
cudaError_t launch_maxabs(const T* Q, int64_t n, int64_t per_tile, int L, int64_t per_elem, int64_t nlocal,
                          unsigned long long* out, int* bad, cudaStream_t s);
size_t local_smem_bytes(int N, int elem_bytes);
size_t sparse_local_smem(int N, int elem_bytes);
size_t sparse_neigh_smem(int N, int elem_bytes);
size_t neigh_smem_bytes(int N, int elem_bytes);
cudaError_t configure_kernels(int N, int elem_bytes);

}  // namespace ydg
