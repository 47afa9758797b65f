// C ABI of libydg.so (include/ydg.h).  Host orchestration: validation, setup, device
// layout, step sequencing (all local updates of a step complete before the
// neighbour flux reads the traces), optional z-slab decomposition with an NCCL halo.
#include "../../include/ydg.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "generated/ydg_counts.h"
#include "generated/ydg_matrices.h"
#include "generic.h"
#include "halo.h"
#include <cstdio>
#include "kernels.cuh"
#include "setup.h"

using namespace ydg;

struct ydg_solver {
  int N = 0, P = 0, prec = 0, dev = 0, B = 0, Bt = 0;
  int status = YDG_OK;  // sticky CUDA / NCCL fault
  std::string err;
  cudaStream_t stream = nullptr;
  // decomposition
  int rank = 0, nranks = 1;
  Halo halo;
  // mesh
  bool have_mesh = false;
  int64_t ne = 0, first = 0, nlocal = 0;
  int64_t nslots = 0;   // local element slots incl. ghosts (multiple of lanes)
  int lanes = 32;       // elements per tile: kDmLanes (fp64 tensor-core kernels) or 32 (fp32)
  int64_t ntiles = 0;   // owned tiles
  Neighbours nbr;       // global tables in internal element numbering
  Neighbours nbr_ext;   // ... in the caller's numbering when the elements are reordered
  int32_t* slot_of = nullptr;  // device: owned external local index -> internal slot (or null)
  // device buffers
  void* Q = nullptr;
  void* traces = nullptr;
  void* traces2 = nullptr;  // fused step kernel: the other trace buffer (steps alternate)
  bool fused = false;       // ydg_step(nsteps >= 2) runs the fused kernel
  void* star = nullptr;
  void* aplus = nullptr;
  void* aminus = nullptr;
  int32_t* nb = nullptr;
  int8_t* jh = nullptr;
  void* staging = nullptr;
  size_t staging_bytes = 0;
  size_t device_bytes = 0;
  int grid_local = 0, grid_neigh = 0;
  int64_t bnd_lo = 0, bnd_hi = 0;  // leading / trailing owned tiles covering all tiles with ghosts
  // generic path (viscoelastic, or YDG_GENERIC=1): canonical layouts, CSR global matrices
  bool generic = false;
  bool visco_tc = false;    // viscoelastic local kernel on FP64 tensor cores (visco.cu)
  void* src = nullptr;      // [e][p][9] viscoelastic source pattern values
  int64_t* nb64 = nullptr;  // [e][4]
  int8_t* jh_e = nullptr;   // [e][4]
  std::vector<void*> csr;   // device CSR arrays (freed in ydg_destroy)
  GenParams gp{};
  // profiling: (start, stop, kind) events of timed launches; kind 0 = local, 1 = neighbour,
  // 2 = fused
  bool profiling = false;
  struct Ev { cudaEvent_t a, b; int kind; };
  std::vector<Ev> pending;
  double prof_ms[3] = {0, 0, 0};  // local, neighbour, fused
  int64_t prof_launches = 0;
  // ydg_step_graph: the launch sequence of (dt, nsteps) captured once into a CUDA graph
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t gexec = nullptr;
  int sims = 1;  // fused simulations (element-simulations v = e * sims + s)
  // two-cluster local time stepping (ydg_set_clusters / ydg_step_lts, reading R26)
  std::vector<int8_t> cluster_ext;  // caller numbering; empty = global time stepping
  bool lts = false;
  int64_t lts_nc = 0;          // coarse elements = internal [0, lts_nc), a multiple of the tile width
  int64_t lts_ncb_tiles = 0;   // tiles covering the coarse elements with a fine neighbour
  int32_t* nb_lts[3] = {nullptr, nullptr, nullptr};  // flux neighbour slots: fine sub 1, fine sub 2, coarse
  int64_t* lts_lst[3] = {nullptr, nullptr, nullptr};  // combine lists: S1 = own, S2 = own - S1, B (=|+=) own
  int64_t lts_n[3] = {0, 0, 0};
  double g_dt = 0;
  int g_n = -1;
  // YDG_GUARD=1 (debug): every mesh/DOF buffer gets kGuard bytes of a fill pattern on both
  // sides; ydg_query(YDG_Q_GUARD_VIOLATIONS) counts overwritten guard bytes (an out-of-bounds
  // store check in place of compute-sanitizer, which this GPU pool does not allow)
  bool guard = false;
  std::vector<std::pair<void*, size_t>> guards;  // user pointer, bytes
};

namespace {

thread_local std::string g_last_error;

int fail(ydg_solver* h, int code, const std::string& msg) {
  h->err = msg;
  if (code == YDG_ERR_CUDA || code == YDG_ERR_NCCL) h->status = code;
  return code;
}

#define CUDA_OR_FAIL(h, call)                                                         \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return fail(h, e_ == cudaErrorMemoryAllocation ? YDG_ERR_OOM : YDG_ERR_CUDA,    \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                \
  } while (0)

int elem_bytes(const ydg_solver* h) { return h->prec; }

// Values per element-face trace block of the fp64 tensor-core kernels (layout
// [tile][face][lane][TS], 16 lanes, block [m][q] padded to 16 bytes); 0 = the fp32 layout
// [tile][face][m][q][32].
int trace_block(const ydg_solver* h) { return h->prec == 8 ? (h->Bt * h->P + 1) / 2 * 2 : 0; }

constexpr size_t kGuard = 64 << 10;
constexpr unsigned char kGuardByte = 0xA5;

void dfree(ydg_solver* h, void* p) {
  if (!p) return;
  for (size_t i = 0; i < h->guards.size(); ++i)
    if (h->guards[i].first == p) {
      cudaFree(static_cast<char*>(p) - kGuard);
      h->guards.erase(h->guards.begin() + static_cast<std::ptrdiff_t>(i));
      return;
    }
  cudaFree(p);
}

void free_mesh(ydg_solver* h) {
  for (void** p : {&h->Q, &h->traces, &h->traces2, &h->star, &h->aplus, &h->aminus, &h->staging, &h->src,
                   reinterpret_cast<void**>(&h->slot_of), reinterpret_cast<void**>(&h->nb_lts[0]),
                   reinterpret_cast<void**>(&h->nb_lts[1]), reinterpret_cast<void**>(&h->nb_lts[2]),
                   reinterpret_cast<void**>(&h->lts_lst[0]), reinterpret_cast<void**>(&h->lts_lst[1]),
                   reinterpret_cast<void**>(&h->lts_lst[2]),
                   reinterpret_cast<void**>(&h->nb), reinterpret_cast<void**>(&h->jh),
                   reinterpret_cast<void**>(&h->nb64), reinterpret_cast<void**>(&h->jh_e)}) {
    dfree(h, *p);
    *p = nullptr;
  }
  h->device_bytes = 0;
  h->have_mesh = false;
  h->lts = false;
  h->fused = false;
  if (h->gexec) cudaGraphExecDestroy(h->gexec);  // captured the old buffers
  h->gexec = nullptr;
  h->g_n = -1;
}

int dalloc(ydg_solver* h, void** p, size_t bytes) {
  const size_t g = h->guard ? kGuard : 0;
  cudaError_t e = cudaMalloc(p, bytes + 2 * g);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *p = nullptr;
    return fail(h, YDG_ERR_OOM, "cudaMalloc of " + std::to_string(bytes) + " bytes failed");
  }
  if (g) {
    char* base = static_cast<char*>(*p);
    e = cudaMemset(base, kGuardByte, g);
    if (e == cudaSuccess) e = cudaMemset(base + g + bytes, kGuardByte, g);
    if (e != cudaSuccess) {
      cudaFree(base);
      *p = nullptr;
      return fail(h, YDG_ERR_CUDA, std::string("guard fill: ") + cudaGetErrorString(e));
    }
    *p = base + g;
    h->guards.emplace_back(*p, bytes);
  }
  h->device_bytes += bytes;
  return YDG_OK;
}

// max |Q| over the owned DOFs (NaN if any is not finite); synchronises the handle's stream.
double max_abs_q(ydg_solver* h) {
  const double nan = std::numeric_limits<double>::quiet_NaN();
  if (!h->have_mesh || !h->Q) return nan;
  void* buf = nullptr;
  if (cudaMalloc(&buf, 16) != cudaSuccess) return nan;
  cudaStream_t s = h->stream;
  cudaError_t e = cudaMemsetAsync(buf, 0, 16, s);
  unsigned long long* out = static_cast<unsigned long long*>(buf);
  int* bad = reinterpret_cast<int*>(out + 1);
  const int64_t PB = static_cast<int64_t>(h->P) * h->B;
  int64_t n, per_tile = 1;
  int L;
  if (h->generic) {  // canonical [e][p][k]
    n = h->nlocal * PB;
    L = 0;
  } else {  // tiled [tile][k][p][L]
    L = h->lanes;
    per_tile = PB * L;
    n = h->ntiles * per_tile;
  }
  if (e == cudaSuccess)
    e = h->prec == 8 ? launch_maxabs<double>(static_cast<const double*>(h->Q), n, per_tile, L, PB, h->nlocal, out, bad, s)
                     : launch_maxabs<float>(static_cast<const float*>(h->Q), n, per_tile, L, PB, h->nlocal, out, bad, s);
  unsigned long long hv[2] = {0, 0};
  if (e == cudaSuccess) e = cudaMemcpyAsync(hv, buf, 16, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(buf);
  if (e != cudaSuccess || static_cast<int>(hv[1] & 0xffffffffu) != 0) return nan;
  double v;
  std::memcpy(&v, &hv[0], sizeof v);
  return v;
}

// Overwritten guard bytes over all guarded buffers (synchronises the device).
int64_t guard_violations(ydg_solver* h) {
  if (cudaDeviceSynchronize() != cudaSuccess) return -2;
  std::vector<unsigned char> buf(kGuard);
  int64_t bad = 0;
  for (const auto& gb : h->guards) {
    const char* p = static_cast<const char*>(gb.first);
    for (const char* src : {p - kGuard, p + gb.second}) {
      if (cudaMemcpy(buf.data(), src, kGuard, cudaMemcpyDeviceToHost) != cudaSuccess) return -2;
      for (unsigned char c : buf) bad += c != kGuardByte;
    }
  }
  return bad;
}

int check(ydg_solver* h) {
  if (!h) return YDG_ERR_ARG;
  if (h->status != YDG_OK) return h->status;
  cudaError_t e = cudaSetDevice(h->dev);
  if (e != cudaSuccess) return fail(h, YDG_ERR_CUDA, cudaGetErrorString(e));
  return YDG_OK;
}

// Per-element coefficients in the tiled layouts of the kernels (tiles of kLanes elements:
// 16 for fp64, 32 for fp32).  fp64 (tensor-core kernels): star [tile][c][p][3][lane] and
// the factored flux solvers [tile][face][12][lane]; fp32 (sparse kernels): star and the
// flux-solver matrices A+-, [tile][face][p][q][lane].
template <typename T>
void pack_tiles(int P, int64_t n, bool factored, int kLanes, const ElementCoeffs& c, std::vector<T>& star,
                std::vector<T>& ap, std::vector<T>& am) {
  for (int64_t t = 0; t < n; ++t) {
    const int64_t tile = t / kLanes, lane = t % kLanes;
    for (int cc = 0; cc < 3; ++cc)
      for (int p = 0; p < P; ++p)
        for (int j = 0; j < 3; ++j)
          star[(((tile * 3 + cc) * P + p) * 3 + j) * kLanes + lane] =
              static_cast<T>(c.star[((t * 3 + cc) * P + p) * 3 + j]);
    if (factored) {
      for (int i = 0; i < 4; ++i)
        for (int k = 0; k < kFaceCoeffs; ++k)
          ap[((tile * 4 + i) * kFaceCoeffs + k) * kLanes + lane] =
              static_cast<T>(c.face[(t * 4 + i) * kFaceCoeffs + k]);
      continue;
    }
    for (int i = 0; i < 4; ++i)
      for (int p = 0; p < P; ++p)
        for (int q = 0; q < P; ++q) {
          const size_t dst = ((((tile * 4 + i) * P + p) * P + q) * kLanes) + lane;
          ap[dst] = static_cast<T>(c.aplus[((t * 4 + i) * P + p) * P + q]);
          am[dst] = static_cast<T>(c.aminus[((t * 4 + i) * P + p) * P + q]);
        }
  }
}

template <typename T>
int upload_coeffs(ydg_solver* h, const double* xyz, const double* material, const double* anel) {
  const int P = h->P;
  const bool factored = sizeof(T) == 8;  // fp64 flux kernel rebuilds A+- from 12 values/face
  const int kLanes = h->lanes;
  const int64_t tiles = h->nslots / kLanes;
  const size_t star_t = static_cast<size_t>(3) * P * 3 * kLanes;  // per tile
  const size_t flux_t = factored ? static_cast<size_t>(4) * kFaceCoeffs * kLanes : static_cast<size_t>(4) * P * P * kLanes;
  int rc;
  if ((rc = dalloc(h, &h->star, tiles * star_t * sizeof(T)))) return rc;
  if ((rc = dalloc(h, &h->aplus, tiles * flux_t * sizeof(T)))) return rc;
  CUDA_OR_FAIL(h, cudaMemset(h->star, 0, tiles * star_t * sizeof(T)));
  CUDA_OR_FAIL(h, cudaMemset(h->aplus, 0, tiles * flux_t * sizeof(T)));
  if (!factored) {
    if ((rc = dalloc(h, &h->aminus, tiles * flux_t * sizeof(T)))) return rc;
    CUDA_OR_FAIL(h, cudaMemset(h->aminus, 0, tiles * flux_t * sizeof(T)));
  }
  // owned elements in chunks of whole tiles
  const int64_t chunk_tiles = 2048;
  std::vector<T> st, ap, am;
  for (int64_t t0 = 0; t0 * kLanes < h->nlocal; t0 += chunk_tiles) {
    const int64_t s0 = t0 * kLanes;
    const int64_t n = std::min<int64_t>(chunk_tiles * kLanes, h->nlocal - s0);
    const int64_t ct = (n + kLanes - 1) / kLanes;
    ElementCoeffs c;
    std::string err;
    if (!element_coeffs(P, h->first + s0, n, xyz, material, anel, h->nbr, &c, &err))
      return fail(h, YDG_ERR_MESH, err);
    st.assign(static_cast<size_t>(ct) * star_t, T(0));
    ap.assign(static_cast<size_t>(ct) * flux_t, T(0));
    am.assign(factored ? 0 : ap.size(), T(0));
    pack_tiles<T>(P, n, factored, kLanes, c, st, ap, am);
    CUDA_OR_FAIL(h, cudaMemcpy(static_cast<T*>(h->star) + static_cast<size_t>(t0) * star_t, st.data(),
                               st.size() * sizeof(T), cudaMemcpyHostToDevice));
    CUDA_OR_FAIL(h, cudaMemcpy(static_cast<T*>(h->aplus) + static_cast<size_t>(t0) * flux_t, ap.data(),
                               ap.size() * sizeof(T), cudaMemcpyHostToDevice));
    if (!factored)
      CUDA_OR_FAIL(h, cudaMemcpy(static_cast<T*>(h->aminus) + static_cast<size_t>(t0) * flux_t, am.data(),
                                 am.size() * sizeof(T), cudaMemcpyHostToDevice));
  }
  return YDG_OK;
}

// Algorithmic HBM bytes per element of each kernel (each array touched once).
// fp64 (tensor-core kernels): local reads Q, star, writes Q and the 4 trace blocks; the
// flux kernel reads Q, own + neighbour trace blocks, the factored flux solvers, writes Q.
// fp32 (sparse kernels): local reads Q, star, writes Q and the 4 traces; the flux kernel
// reads Q, A+ and A-, own + neighbour traces, writes Q (both flux terms, one lift per face).
double alg_bytes_local(const ydg_solver* h) {
  const double P = h->P, B = h->B, Bt = h->Bt;
  if (h->prec == 8) return (2 * B * P + 3 * P * 3 + 4 * trace_block(h)) * elem_bytes(h);
  return (2 * B * P + 3 * P * 3 + 4 * Bt * P) * elem_bytes(h);
}
double alg_bytes_neigh(const ydg_solver* h) {
  const double P = h->P, B = h->B, Bt = h->Bt;
  if (h->prec == 8) return (2 * B * P + 4 * kFaceCoeffs + 2 * 4 * trace_block(h)) * elem_bytes(h) + 4 * (4 + 1);
  return (2 * B * P + 2 * 4 * P * P + 2 * 4 * Bt * P) * elem_bytes(h) + 4 * (4 + 1);
}
// the tiled elastic kernels (fp64 and fp32) lift the local + neighbour flux once per face
bool shared_lift(const ydg_solver* h) { return h->prec == 8 || !h->generic; }

// fused kernel (fp64): Q read and written once, star, the 4 trace blocks written, own and
// neighbour trace blocks read, the factored flux solvers, neighbour slots and j|h
double alg_bytes_fused(const ydg_solver* h) {
  const double P = h->P, B = h->B;
  return (2 * B * P + 3 * P * 3 + 4 * kFaceCoeffs + 3 * 4 * trace_block(h)) * elem_bytes(h) + 4 * (4 + 1);
}

// Wrap a launch with CUDA events when profiling.
template <typename F>
cudaError_t timed(ydg_solver* h, int kind, cudaStream_t s, F&& launch) {
  if (!h->profiling) return launch();
  ydg_solver::Ev ev{nullptr, nullptr, kind};
  cudaError_t e = cudaEventCreate(&ev.a);
  if (e == cudaSuccess) e = cudaEventCreate(&ev.b);
  if (e == cudaSuccess) e = cudaEventRecord(ev.a, s);
  if (e == cudaSuccess) e = launch();
  if (e == cudaSuccess) e = cudaEventRecord(ev.b, s);
  if (e == cudaSuccess) h->pending.push_back(ev);
  return e;
}

int drain_profile(ydg_solver* h) {
  for (auto& ev : h->pending) {
    float ms = 0;
    CUDA_OR_FAIL(h, cudaEventSynchronize(ev.b));
    CUDA_OR_FAIL(h, cudaEventElapsedTime(&ms, ev.a, ev.b));
    h->prof_ms[ev.kind] += ms;
    h->prof_launches++;
    cudaEventDestroy(ev.a);
    cudaEventDestroy(ev.b);
  }
  h->pending.clear();
  return YDG_OK;
}

template <typename T>
int do_step(ydg_solver* h, double dt, int nsteps, cudaStream_t s) {
  StepParams<T> prm{};
  prm.Q = static_cast<T*>(h->Q);
  prm.traces = static_cast<T*>(h->traces);
  prm.star = static_cast<const T*>(h->star);
  prm.aplus = static_cast<const T*>(h->aplus);
  prm.aminus = static_cast<const T*>(h->aminus);
  prm.nb = h->nb;
  prm.jh = h->jh;
  prm.dt = static_cast<T>(dt);
  for (int d = 0; d < h->N; ++d) {
    prm.scal[d] = static_cast<T>(dt / (d + 1));
    prm.scal[h->N + d] = static_cast<T>(dt / (d + 2));
  }
  if constexpr (sizeof(T) == 8) {
    if (h->fused && h->nranks == 1 && nsteps >= 2) {
      // local(0) -> traces A; fused(n) = flux of step n-1 from one buffer + local(n) into the
      // other; flux of the last step
      T* tb[2] = {static_cast<T*>(h->traces), static_cast<T*>(h->traces2)};
      prm.tile0 = 0;
      prm.ntiles = h->ntiles;
      const int gl = static_cast<int>(std::min<int64_t>(h->grid_local, prm.ntiles));
      prm.traces = tb[0];
      CUDA_OR_FAIL(h, timed(h, 0, s, [&] { return launch_local<T>(h->N, prm, gl, s); }));
      for (int n = 1; n < nsteps; ++n) {
        prm.traces_in = tb[(n - 1) & 1];
        prm.traces = tb[n & 1];
        CUDA_OR_FAIL(h, timed(h, 2, s, [&] { return launch_fused(h->N, prm, gl, s); }));
      }
      prm.traces = tb[(nsteps - 1) & 1];
      prm.traces_in = nullptr;
      const int64_t units = prm.ntiles * (h->lanes / 8);
      CUDA_OR_FAIL(h, timed(h, 1, s, [&] { return launch_neigh<T>(h->N, prm, static_cast<int>(std::min<int64_t>(h->grid_neigh, units)), s); }));
      return YDG_OK;
    }
  }
  for (int n = 0; n < nsteps; ++n) {
    if (h->nranks > 1) {
      // boundary tiles first, then send their traces while the interior proceeds
      auto local = [&](int64_t t0, int64_t n) -> int {
        if (n <= 0) return YDG_OK;
        prm.tile0 = t0;
        prm.ntiles = n;
        CUDA_OR_FAIL(h, timed(h, 0, s, [&] { return launch_local<T>(h->N, prm, static_cast<int>(std::min<int64_t>(h->grid_local, n)), s); }));
        return YDG_OK;
      };
      int rc = local(0, h->bnd_lo);
      if (!rc) rc = local(h->ntiles - h->bnd_hi, h->bnd_hi);
      if (rc) return rc;
      rc = h->halo.exchange(s, h->traces, elem_bytes(h), &h->err);
      if (rc) return fail(h, rc, h->err);
      if ((rc = local(h->bnd_lo, h->ntiles - h->bnd_hi - h->bnd_lo))) return rc;
      rc = h->halo.wait(s, &h->err);
      if (rc) return fail(h, rc, h->err);
    } else {
      prm.tile0 = 0;
      prm.ntiles = h->ntiles;
      CUDA_OR_FAIL(h, timed(h, 0, s, [&] { return launch_local<T>(h->N, prm, static_cast<int>(std::min<int64_t>(h->grid_local, prm.ntiles)), s); }));
    }
    prm.tile0 = 0;
    prm.ntiles = h->ntiles;
    const int64_t units = prm.ntiles * (h->prec == 8 ? h->lanes / 8 : 1);  // fp64 flux CTAs take 8-element halves
    CUDA_OR_FAIL(h, timed(h, 1, s, [&] { return launch_neigh<T>(h->N, prm, static_cast<int>(std::min<int64_t>(h->grid_neigh, units)), s); }));
  }
  return YDG_OK;
}

cudaStream_t pick_stream(ydg_solver* h, void* s) { return s ? static_cast<cudaStream_t>(s) : h->stream; }

// ---------------------------------------------------------------- generic path

// Column patterns: star-matrix rows (setup.cpp star_cols) and viscoelastic source rows
// (reading R14: E[sigma_s][theta^l_t] for t normal when s normal, t = s when s shear;
// E[theta^l_s][theta^l_s]; velocity rows have no source).  Unused slots repeat a column
// with a zero coefficient.
void generic_patterns(int P, int (*ecols)[9], int (*scols)[3]) {
  for (int p = 0; p < 27; ++p) {
    star_cols(P, p < P ? p : p % 9, scols[p]);  // the layout element_coeffs uploads for P
    int n = 0;
    if (p < 6) {
      for (int l = 0; l < 3; ++l)
        for (int t = 0; t < 6; ++t)
          if ((p < 3 && t < 3) || p == t) ecols[p][n++] = 9 + 6 * l + t;
    } else if (p >= 9) {
      ecols[p][n++] = p;
    }
    const int fill = n ? ecols[p][0] : 0;
    while (n < 9) ecols[p][n++] = fill;
  }
}

template <class TB>
void csr_from(int rows, int cols, const std::function<double(int, int)>& at, std::vector<int>& ptr,
              std::vector<int>& col, std::vector<double>& val) {
  (void)sizeof(TB);
  ptr.assign(1, 0);
  col.clear();
  val.clear();
  for (int r = 0; r < rows; ++r) {
    for (int c = 0; c < cols; ++c) {
      const double v = at(r, c);
      if (v != 0.0) {
        col.push_back(c);
        val.push_back(v);
      }
    }
    ptr.push_back(static_cast<int>(col.size()));
  }
}

template <class TB>
int upload_csr(ydg_solver* h) {
  constexpr int B = TB::B, Bt = TB::Bt;
  struct M { int rows, cols; std::function<double(int, int)> at; const int** ptr; const int** col; const double** val; };
  GenParams& g = h->gp;
  std::vector<M> ms = {
      {3 * B, B, [](int r, int c) { return -kdir(TB::K, r / B, c, r % B); }, &g.kt_ptr, &g.kt_col, &g.kt_val},
      {3 * B, B, [](int r, int c) { return kdir(TB::K, r / B, r % B, c); }, &g.kh_ptr, &g.kh_col, &g.kh_val},
      {4 * Bt, B, [](int r, int c) { return TB::R[r / Bt][c][r % Bt]; }, &g.rt_ptr, &g.rt_col, &g.rt_val},
      {4 * B, Bt, [](int r, int c) { return TB::R[r / B][r % B][c]; }, &g.r_ptr, &g.r_col, &g.r_val},
      {3 * Bt, Bt, [](int r, int c) { return TB::f[r / Bt][r % Bt][c]; }, &g.f_ptr, &g.f_col, &g.f_val}};
  for (auto& m : ms) {
    std::vector<int> ptr, col;
    std::vector<double> val;
    csr_from<TB>(m.rows, m.cols, m.at, ptr, col, val);
    void *dp = nullptr, *dc = nullptr, *dv = nullptr;
    if (cudaMalloc(&dp, ptr.size() * sizeof(int)) != cudaSuccess ||
        cudaMalloc(&dc, std::max<size_t>(1, col.size()) * sizeof(int)) != cudaSuccess ||
        cudaMalloc(&dv, std::max<size_t>(1, val.size()) * sizeof(double)) != cudaSuccess)
      return fail(h, YDG_ERR_OOM, "CSR allocation failed");
    h->csr.insert(h->csr.end(), {dp, dc, dv});
    CUDA_OR_FAIL(h, cudaMemcpy(dp, ptr.data(), ptr.size() * sizeof(int), cudaMemcpyHostToDevice));
    if (!col.empty()) {
      CUDA_OR_FAIL(h, cudaMemcpy(dc, col.data(), col.size() * sizeof(int), cudaMemcpyHostToDevice));
      CUDA_OR_FAIL(h, cudaMemcpy(dv, val.data(), val.size() * sizeof(double), cudaMemcpyHostToDevice));
    }
    *m.ptr = static_cast<const int*>(dp);
    *m.col = static_cast<const int*>(dc);
    *m.val = static_cast<const double*>(dv);
    if (m.ptr == &g.kt_ptr) g.kt_nnz = static_cast<int>(val.size());
    if (m.ptr == &g.kh_ptr) g.kh_nnz = static_cast<int>(val.size());
  }
  return YDG_OK;
}

int generic_matrices(ydg_solver* h) {
  switch (h->N) {
    case 1: return upload_csr<tables::N1>(h);
    case 2: return upload_csr<tables::N2>(h);
    case 3: return upload_csr<tables::N3>(h);
    case 4: return upload_csr<tables::N4>(h);
    case 5: return upload_csr<tables::N5>(h);
    case 6: return upload_csr<tables::N6>(h);
  }
  return fail(h, YDG_ERR_UNSUPPORTED, "order not tabulated");
}

// Mesh upload of the generic path: element-major layouts (generic.h), one rank.
int generic_upload_mesh(ydg_solver* h, const double* xyz, const double* material, const double* anel) {
  const int P = h->P, B = h->B, Bt = h->Bt;
  const int64_t ne = h->ne;
  int rc;
  if ((rc = dalloc(h, &h->Q, static_cast<size_t>(ne) * P * B * 8))) return rc;
  if ((rc = dalloc(h, &h->traces, static_cast<size_t>(ne) * 4 * Bt * 9 * 8))) return rc;
  if ((rc = dalloc(h, &h->star, static_cast<size_t>(ne) * 3 * P * 3 * 8))) return rc;
  if ((rc = dalloc(h, &h->aplus, static_cast<size_t>(ne) * 4 * P * 9 * 8))) return rc;
  if ((rc = dalloc(h, &h->aminus, static_cast<size_t>(ne) * 4 * P * 9 * 8))) return rc;
  if ((rc = dalloc(h, reinterpret_cast<void**>(&h->nb64), static_cast<size_t>(ne) * 4 * 8))) return rc;
  if ((rc = dalloc(h, reinterpret_cast<void**>(&h->jh_e), static_cast<size_t>(ne) * 4))) return rc;
  if (P == 27 && (rc = dalloc(h, &h->src, static_cast<size_t>(ne) * P * 9 * 8))) return rc;
  CUDA_OR_FAIL(h, cudaMemset(h->Q, 0, static_cast<size_t>(ne) * P * B * 8));
  CUDA_OR_FAIL(h, cudaMemcpy(h->nb64, h->nbr.nb.data(), ne * 4 * 8, cudaMemcpyHostToDevice));
  {
    std::vector<int8_t> jh(ne * 4);
    for (int64_t i = 0; i < ne * 4; ++i) jh[i] = static_cast<int8_t>(h->nbr.j[i] | (h->nbr.h[i] << 2));
    CUDA_OR_FAIL(h, cudaMemcpy(h->jh_e, jh.data(), jh.size(), cudaMemcpyHostToDevice));
  }
  int ecols[27][9], scols[27][3];
  generic_patterns(P, ecols, scols);
  if (P == 27) {
    if (!(anel[0] > 0.0) || !std::isfinite(anel[0])) h->visco_tc = false;
    for (int l = 0; l < 3; ++l) h->gp.wratio[l] = h->visco_tc ? anel[l] / anel[0] : 1.0;
  }
  const int64_t chunk = 65536;
  std::vector<double> st, ap, am, sr;
  for (int64_t e0 = 0; e0 < ne; e0 += chunk) {
    const int64_t n = std::min(chunk, ne - e0);
    ElementCoeffs c;
    std::string err;
    if (!element_coeffs(P, e0, n, xyz, material, anel, h->nbr, &c, &err)) return fail(h, YDG_ERR_MESH, err);
    ap.assign(n * 4 * P * 9, 0.0);
    am.assign(ap.size(), 0.0);
    for (int64_t t = 0; t < n; ++t)
      for (int i = 0; i < 4; ++i)
        for (int p = 0; p < P; ++p)
          for (int q = 0; q < P; ++q) {
            const double vp = c.aplus[((t * 4 + i) * P + p) * P + q], vm = c.aminus[((t * 4 + i) * P + p) * P + q];
            if (q < 9) {
              ap[((t * 4 + i) * P + p) * 9 + q] = vp;
              am[((t * 4 + i) * P + p) * 9 + q] = vm;
            } else if (vp != 0.0 || vm != 0.0) {
              return fail(h, YDG_ERR_MESH, "flux solver couples a memory variable (unexpected)");
            }
          }
    if (P == 27 && h->visco_tc) {  // the tensor-core kernel scales mechanism 0's memory-variable rows
      for (int64_t t = 0; t < n && h->visco_tc; ++t)
        for (int cc = 0; cc < 3; ++cc)
          for (int sv = 0; sv < 6; ++sv)
            for (int l = 1; l < 3; ++l)
              for (int k = 0; k < 3; ++k) {
                const double b = c.star[((t * 3 + cc) * P + 9 + sv) * 3 + k];
                const double v = c.star[((t * 3 + cc) * P + 9 + 6 * l + sv) * 3 + k];
                if (std::fabs(v - h->gp.wratio[l] * b) > 1e-13 * (std::fabs(v) + std::fabs(b)) + 1e-300)
                  h->visco_tc = false;  // not proportional: the CSR kernels take over
              }
    }
    CUDA_OR_FAIL(h, cudaMemcpy(static_cast<double*>(h->star) + e0 * 3 * P * 3, c.star.data(), c.star.size() * 8,
                               cudaMemcpyHostToDevice));
    CUDA_OR_FAIL(h, cudaMemcpy(static_cast<double*>(h->aplus) + e0 * 4 * P * 9, ap.data(), ap.size() * 8,
                               cudaMemcpyHostToDevice));
    CUDA_OR_FAIL(h, cudaMemcpy(static_cast<double*>(h->aminus) + e0 * 4 * P * 9, am.data(), am.size() * 8,
                               cudaMemcpyHostToDevice));
    if (P == 27) {
      sr.assign(n * P * 9, 0.0);
      for (int64_t t = 0; t < n; ++t)
        for (int p = 0; p < P; ++p) {
          bool seen[27] = {};
          for (int j = 0; j < 9; ++j) {
            const int q = ecols[p][j];
            if (seen[q]) continue;  // padding slot repeats a column with a zero value
            seen[q] = true;
            sr[(t * P + p) * 9 + j] = c.src[(t * P + p) * P + q];
          }
        }
      CUDA_OR_FAIL(h, cudaMemcpy(static_cast<double*>(h->src) + e0 * P * 9, sr.data(), sr.size() * 8,
                                 cudaMemcpyHostToDevice));
    }
  }
  GenParams& g = h->gp;
  g.Q = static_cast<double*>(h->Q);
  g.traces = static_cast<double*>(h->traces);
  g.star = static_cast<const double*>(h->star);
  g.src = static_cast<const double*>(h->src);
  g.aplus = static_cast<const double*>(h->aplus);
  g.aminus = static_cast<const double*>(h->aminus);
  g.nb = h->nb64;
  g.jh = h->jh_e;
  g.N = h->N;
  g.B = B;
  g.Bt = Bt;
  g.P = P;
  h->nslots = ne;
  h->ntiles = (ne + kLanes - 1) / kLanes;
  return YDG_OK;
}

int generic_step(ydg_solver* h, double dt, int nsteps, cudaStream_t s) {
  GenParams g = h->gp;
  g.dt = dt;
  for (int d = 0; d < h->N; ++d) {
    g.scal[d] = dt / (d + 1);
    g.scal[h->N + d] = dt / (d + 2);
  }
  g.e0 = 0;
  g.n = h->ne;
  for (int n = 0; n < nsteps; ++n) {
    CUDA_OR_FAIL(h, timed(h, 0, s, [&] { return h->visco_tc ? visco_launch_local(g, s) : gen_launch(g, true, s); }));
    CUDA_OR_FAIL(h, timed(h, 1, s, [&] { return h->visco_tc ? visco_launch_neigh(g, s) : gen_launch(g, false, s); }));
  }
  return YDG_OK;
}

}  // namespace

extern "C" {

const char* ydg_last_error(void) { return g_last_error.c_str(); }

int ydg_create(int order, int quantities, int precision, int cuda_device, ydg_solver** out) {
  if (!out) return YDG_ERR_ARG;
  *out = nullptr;
  if (order < 1 || order > kMaxN || (quantities != 9 && quantities != 27) ||
      (precision != 4 && precision != 8)) {
    g_last_error = "bad order / quantities / precision";
    return YDG_ERR_ARG;
  }
  const char* force = std::getenv("YDG_GENERIC");
  const bool generic = quantities == 27 || (order == 6 && precision == 8) || (force && force[0] == '1');
  if (generic && precision != 8) {
    g_last_error = "the generic (viscoelastic) path is fp64 only";
    return YDG_ERR_UNSUPPORTED;
  }
  if (generic && gen_local_te((order + 1) * (order + 2) * (order + 3) / 6, (order + 1) * (order + 2) / 2, quantities) == 0) {
    g_last_error = "the generic kernel's work arrays exceed the shared memory of a CTA";
    return YDG_ERR_UNSUPPORTED;
  }
  std::unique_ptr<ydg_solver> h(new ydg_solver);
  h->N = order;
  h->P = quantities;
  h->prec = precision;
  h->dev = cuda_device;
  h->B = (order + 1) * (order + 2) * (order + 3) / 6;
  h->Bt = (order + 1) * (order + 2) / 2;
  h->generic = generic;
  const char* gv = std::getenv("YDG_GUARD");
  h->guard = gv && gv[0] == '1';
  cudaError_t e = cudaSetDevice(cuda_device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) {
    if (generic) {
      int ecols[27][9], scols[27][3];
      generic_patterns(quantities, ecols, scols);
      e = gen_configure(h->B, h->Bt, quantities, ecols, scols);
      const char* vg = std::getenv("YDG_VISCO_GENERIC");  // 1: CSR local kernel (comparison)
      h->visco_tc = visco_supported(order, quantities) && !(vg && vg[0] == '1');
      if (e == cudaSuccess && h->visco_tc) e = visco_configure(order, scols);
    } else {
      e = configure_kernels(order, precision);
    }
  }
  if (e != cudaSuccess) {
    g_last_error = std::string("CUDA: ") + cudaGetErrorString(e);
    return YDG_ERR_CUDA;
  }
  if (generic) {
    int rc = generic_matrices(h.get());
    if (rc) {
      g_last_error = h->err;
      for (void* p : h->csr) cudaFree(p);
      return rc;
    }
  }
  *out = h.release();
  return YDG_OK;
}

int ydg_set_comm(ydg_solver* h, int rank, int nranks, const void* nccl_unique_id) {
  int rc = check(h);
  if (rc) return rc;
  if (h->have_mesh) return fail(h, YDG_ERR_STATE, "ydg_set_comm must precede ydg_upload_mesh");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(h, YDG_ERR_ARG, "bad rank / nranks");
  if (nranks > 1 && !nccl_unique_id) return fail(h, YDG_ERR_ARG, "null NCCL unique id");
  h->rank = rank;
  h->nranks = nranks;
  if (nranks > 1) {
    rc = h->halo.init(rank, nranks, nccl_unique_id, &h->err);
    if (rc) return fail(h, rc, h->err);
  }
  return YDG_OK;
}

int ydg_set_simulations(ydg_solver* h, int S) {
  int rc = check(h);
  if (rc) return rc;
  if (h->have_mesh) return fail(h, YDG_ERR_STATE, "ydg_set_simulations must precede ydg_upload_mesh");
  if (S < 1 || S > 64) return fail(h, YDG_ERR_ARG, "simulations must be in [1, 64]");
  h->sims = S;
  return YDG_OK;
}

static int upload_mesh_impl(ydg_solver* h, int64_t ne, const double* xyz, const int64_t* vid,
                            const double* material, const double* anelastic);
static int upload_tiled(ydg_solver* h, const double* xyz, const double* material, const double* anelastic);

int ydg_upload_mesh(ydg_solver* h, int64_t ne, const double* xyz, const int64_t* vid,
                    const double* material, const double* anelastic) {
  int rc = check(h);
  if (rc) return rc;
  if (ne <= 0 || !xyz || !vid || !material) return fail(h, YDG_ERR_ARG, "null mesh input or ne <= 0");
  if (h->sims == 1) return upload_mesh_impl(h, ne, xyz, vid, material, anelastic);
  // fused simulations: element-simulation v = e * S + s carries element e's geometry and
  // material; the vertex ids of simulation s are shifted by s * (max id + 1), so faces match
  // within a simulation only and Neigh(v, i) = Neigh(e, i) * S + s
  const int64_t S = h->sims, nv = ne * S;
  int64_t vmax = 0;
  for (int64_t i = 0; i < ne * 4; ++i) vmax = std::max(vmax, vid[i]);
  std::vector<double> xyz_v(static_cast<size_t>(nv) * 12), mat_v(static_cast<size_t>(nv) * 3);
  std::vector<int64_t> vid_v(static_cast<size_t>(nv) * 4);
  std::vector<double> an_v;
  if (anelastic) an_v.assign(anelastic, anelastic + 3), an_v.resize(3 + static_cast<size_t>(nv) * 6);
  for (int64_t e = 0; e < ne; ++e)
    for (int64_t sm = 0; sm < S; ++sm) {
      const int64_t v = e * S + sm;
      std::copy(xyz + e * 12, xyz + e * 12 + 12, xyz_v.begin() + v * 12);
      std::copy(material + e * 3, material + e * 3 + 3, mat_v.begin() + v * 3);
      for (int k = 0; k < 4; ++k) vid_v[v * 4 + k] = vid[e * 4 + k] + sm * (vmax + 1);
      if (anelastic) std::copy(anelastic + 3 + e * 6, anelastic + 9 + e * 6, an_v.begin() + 3 + v * 6);
    }
  return upload_mesh_impl(h, nv, xyz_v.data(), vid_v.data(), mat_v.data(), anelastic ? an_v.data() : nullptr);
}

// Internal element order of the tiled paths (see upload_mesh_impl): ext_of[i] = caller id of
// internal element i.  Each rank range [r ne / R, (r+1) ne / R) is permuted within itself
// (so every rank derives the same global numbering): elements with a neighbour in another
// range first, then ascending Morton code of the centroid (21 bits per axis over the bounding
// box of all centroids), ties by caller id.
static std::vector<int64_t> locality_order(int64_t ne, const double* xyz, const Neighbours& nbr, int nranks) {
  std::vector<double> c(static_cast<size_t>(ne) * 3);
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int64_t e = 0; e < ne; ++e)
    for (int d = 0; d < 3; ++d) {
      const double* x = xyz + e * 12;
      const double v = 0.25 * (x[d] + x[3 + d] + x[6 + d] + x[9 + d]);
      c[e * 3 + d] = v;
      lo[d] = std::min(lo[d], v);
      hi[d] = std::max(hi[d], v);
    }
  auto spread = [](uint64_t v) {  // 21 bits -> every third bit
    v &= 0x1fffff;
    v = (v | v << 32) & 0x1f00000000ffffULL;
    v = (v | v << 16) & 0x1f0000ff0000ffULL;
    v = (v | v << 8) & 0x100f00f00f00f00fULL;
    v = (v | v << 4) & 0x10c30c30c30c30c3ULL;
    v = (v | v << 2) & 0x1249249249249249ULL;
    return v;
  };
  std::vector<uint64_t> key(static_cast<size_t>(ne));
  for (int64_t e = 0; e < ne; ++e) {
    uint64_t m = 0;
    for (int d = 0; d < 3; ++d) {
      const double span = hi[d] > lo[d] ? hi[d] - lo[d] : 1.0;
      const uint64_t q = static_cast<uint64_t>((c[e * 3 + d] - lo[d]) / span * 2097151.0);
      m |= spread(q) << d;
    }
    key[e] = m;
  }
  std::vector<int64_t> ext_of(static_cast<size_t>(ne));
  for (int r = 0; r < nranks; ++r) {
    const int64_t a = ne * r / nranks, b = ne * (r + 1) / nranks;
    std::vector<std::pair<std::pair<int, uint64_t>, int64_t>> k;
    k.reserve(static_cast<size_t>(b - a));
    for (int64_t e = a; e < b; ++e) {
      int bnd = 0;
      for (int i = 0; i < 4; ++i) {
        const int64_t n = nbr.nb[e * 4 + i];
        bnd |= (n < a || n >= b);
      }
      k.push_back({{bnd ? 0 : 1, key[e]}, e});
    }
    std::sort(k.begin(), k.end());
    for (int64_t i = a; i < b; ++i) ext_of[i] = k[i - a].second;
  }
  return ext_of;
}

static int upload_mesh_impl(ydg_solver* h, int64_t ne, const double* xyz, const int64_t* vid,
                            const double* material, const double* anelastic) {
  int rc = 0;
  if (h->P == 27 && !anelastic) return fail(h, YDG_ERR_ARG, "viscoelastic solver needs anelastic data");
  for (int64_t e = 0; e < ne; ++e) {
    const double* m = material + e * 3;
    if (!(m[0] > 0 && m[1] > 0 && m[2] > 0 && m[1] > m[2]))
      return fail(h, YDG_ERR_ARG, "material must satisfy rho > 0, vp > vs > 0");
  }
  Neighbours nbr;
  std::string err;
  if (!match_faces(ne, vid, &nbr, &err)) return fail(h, YDG_ERR_MESH, err);
  free_mesh(h);
  h->ne = ne;
  h->first = ne * h->rank / h->nranks;
  h->nlocal = ne * (h->rank + 1) / h->nranks - h->first;
  // Optional locality reordering of the tiled (fp64 / fp32 elastic) paths (YDG_REORDER=1):
  // within every rank's element range, elements with an off-rank neighbour first (they are
  // launched before the halo), then by the Morton code of their centroid, so that the
  // neighbour traces a flux tile gathers were written by nearby tiles.  Internal numbering
  // only: the DOF calls, ydg_get_neighbours and the rank ranges use the caller's ids.
  // Measured on c1 / c2: flux 7.90 -> 7.87 ms, fp32 ader_neigh 23.9 -> 25.6 ms,
  // so it is off by default (the kernels are latency-, not DRAM-bound).
  std::vector<int64_t> ext_of;
  const char* ro = std::getenv("YDG_REORDER");
  if (!h->cluster_ext.empty()) {
    // LTS: coarse elements with a fine neighbour, the other coarse elements, then the fine
    // ones (caller order within each class), so that every launch of a cycle covers one
    // contiguous tile range
    if (h->generic || h->prec != 8 || h->nranks > 1)
      return fail(h, YDG_ERR_UNSUPPORTED, "local time stepping runs on the fp64 elastic tensor-core path, one rank");
    if (static_cast<int64_t>(h->cluster_ext.size()) != ne) return fail(h, YDG_ERR_ARG, "cluster array size != elements");
    std::vector<int64_t> cb, ci, fi;
    for (int64_t e = 0; e < ne; ++e) {
      if (h->cluster_ext[e] == 0) { fi.push_back(e); continue; }
      bool bnd = false;
      for (int i = 0; i < 4; ++i) bnd |= h->cluster_ext[nbr.nb[e * 4 + i]] == 0;
      (bnd ? cb : ci).push_back(e);
    }
    const int64_t nc = static_cast<int64_t>(cb.size() + ci.size());
    if (nc % kDmLanes) return fail(h, YDG_ERR_ARG, "the coarse cluster must hold a multiple of the tile width (YDG_Q_TILE_ELEMENTS)");
    ext_of = cb;
    ext_of.insert(ext_of.end(), ci.begin(), ci.end());
    ext_of.insert(ext_of.end(), fi.begin(), fi.end());
    h->lts = true;
    h->lts_nc = nc;
    h->lts_ncb_tiles = (static_cast<int64_t>(cb.size()) + kDmLanes - 1) / kDmLanes;
  } else if (!h->generic && ro && ro[0] == '1') {
    ext_of = locality_order(ne, xyz, nbr, h->nranks);
  }
  if (!ext_of.empty()) {  // internal numbering = ext_of
    std::vector<double> xyz_i(static_cast<size_t>(ne) * 12), mat_i(static_cast<size_t>(ne) * 3);
    std::vector<int64_t> vid_i(static_cast<size_t>(ne) * 4);
    for (int64_t i = 0; i < ne; ++i) {
      const int64_t e = ext_of[i];
      std::copy(xyz + e * 12, xyz + e * 12 + 12, xyz_i.begin() + i * 12);
      std::copy(material + e * 3, material + e * 3 + 3, mat_i.begin() + i * 3);
      std::copy(vid + e * 4, vid + e * 4 + 4, vid_i.begin() + i * 4);
    }
    Neighbours nbr_i;
    if (!match_faces(ne, vid_i.data(), &nbr_i, &err)) return fail(h, YDG_ERR_MESH, err);
    h->nbr_ext = std::move(nbr);
    h->nbr = std::move(nbr_i);
    std::vector<int32_t> slot(static_cast<size_t>(h->nlocal));
    for (int64_t i = h->first; i < h->first + h->nlocal; ++i) slot[ext_of[i] - h->first] = static_cast<int32_t>(i - h->first);
    if ((rc = dalloc(h, reinterpret_cast<void**>(&h->slot_of), slot.size() * sizeof(int32_t)))) { free_mesh(h); return rc; }
    CUDA_OR_FAIL(h, cudaMemcpy(h->slot_of, slot.data(), slot.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    return upload_tiled(h, xyz_i.data(), mat_i.data(), anelastic);
  }
  h->nbr = std::move(nbr);
  h->nbr_ext = Neighbours();
  if (h->generic) {
    if (h->nranks > 1) return fail(h, YDG_ERR_UNSUPPORTED, "the generic (viscoelastic) path runs on one rank");
    rc = generic_upload_mesh(h, xyz, material, anelastic);
    if (rc) { free_mesh(h); return rc; }
    h->have_mesh = true;
    return YDG_OK;
  }
  return upload_tiled(h, xyz, material, anelastic);
}

// Device layout of the tiled paths, for the elements in internal numbering (h->nbr).
static int upload_tiled(ydg_solver* h, const double* xyz, const double* material, const double* anelastic) {
  int rc = 0;
  h->lanes = h->prec == 8 ? kDmLanes : 32;
  const int kLanes = h->lanes;
  h->ntiles = (h->nlocal + kLanes - 1) / kLanes;
  // local slots: owned [0, nlocal) padded to tiles, then ghosts
  std::vector<int64_t> ghost_of;  // global element id of each ghost slot
  std::vector<int32_t> nb_local(static_cast<size_t>(h->ntiles) * kLanes * 4, 0);
  // j | h << 2 per (tile, face): kLanes bytes, padded to 16 (TMA granularity) for fp64 tiles
  const int jh_stride = kLanes < 16 ? 16 : kLanes;
  std::vector<int8_t> jh_local(static_cast<size_t>(h->ntiles) * 4 * jh_stride, 0);
  int64_t owned_slots = h->ntiles * kLanes;
  std::vector<int64_t> boundary;  // owned tiles with ghosts
  if (h->nranks > 1) {
    rc = h->halo.plan(h->nbr, h->first, h->nlocal, owned_slots, &ghost_of, &h->err);
    if (rc) return fail(h, rc, h->err);
  }
  h->nslots = owned_slots + static_cast<int64_t>((ghost_of.size() + kLanes - 1) / kLanes) * kLanes;
  {
    // map global neighbour ids to local slots
    std::vector<std::pair<int64_t, int64_t>> gmap(ghost_of.size());
    for (size_t g = 0; g < ghost_of.size(); ++g) gmap[g] = {ghost_of[g], owned_slots + static_cast<int64_t>(g)};
    std::sort(gmap.begin(), gmap.end());
    std::vector<char> is_boundary(h->ntiles, 0);
    for (int64_t l = 0; l < h->ntiles * kLanes; ++l) {
      const int64_t tile = l / kLanes, lane = l % kLanes;
      for (int i = 0; i < 4; ++i) {
        const size_t dst = (tile * 4 + i) * kLanes + lane;
        if (l >= h->nlocal) {  // padding lane: points to itself, zero data
          nb_local[dst] = static_cast<int32_t>(l);
          continue;
        }
        const int64_t g = h->first + l;
        const int64_t n = h->nbr.nb[g * 4 + i];
        int64_t slot;
        if (n >= h->first && n < h->first + h->nlocal) {
          slot = n - h->first;
        } else {
          auto it = std::lower_bound(gmap.begin(), gmap.end(), std::make_pair(n, int64_t(-1)));
          if (it == gmap.end() || it->first != n) return fail(h, YDG_ERR_MESH, "ghost map incomplete");
          slot = it->second;
          is_boundary[tile] = 1;
        }
        if (slot > INT32_MAX) return fail(h, YDG_ERR_UNSUPPORTED, "more than 2^31 local elements");
        nb_local[dst] = static_cast<int32_t>(slot);
        jh_local[(tile * 4 + i) * jh_stride + lane] = static_cast<int8_t>(h->nbr.j[g * 4 + i] | (h->nbr.h[g * 4 + i] << 2));
      }
    }
    // Tiles with ghost neighbours are launched before the interior so their traces can be
    // sent while the interior computes.  With z-major element order a slab's boundary
    // tiles sit at both ends of its range: [0, bnd_lo) and [ntiles - bnd_hi, ntiles)
    // cover every tile with a ghost (for other orders these ranges simply grow).
    h->bnd_lo = h->bnd_hi = 0;
    const int64_t half = h->ntiles / 2;
    const bool reordered = !h->nbr_ext.nb.empty();  // locality order: boundary elements first
    for (int64_t t = 0; t < h->ntiles; ++t)
      if (is_boundary[t]) {
        if (t < half || reordered) h->bnd_lo = std::max(h->bnd_lo, t + 1);
        else h->bnd_hi = std::max(h->bnd_hi, h->ntiles - t);
      }
  }
  // LTS: extra trace slots after the owned ones -- S1, S2 (the coarse element's traces of
  // I over [0, dt] and [dt, 2 dt]) per coarse element with a fine neighbour, B (the sum of
  // the two fine substeps' traces) per fine element with a coarse neighbour -- and the
  // neighbour-slot tables of the three flux launches of a cycle
  std::vector<int32_t> nbt[3];
  std::vector<int64_t> lst[3];
  if (h->lts) {
    const int64_t nc = h->lts_nc;
    std::vector<int64_t> s1(h->nlocal, -1), bslot(h->nlocal, -1);
    int64_t next = h->nslots;
    for (int64_t e = 0; e < h->nlocal; ++e) {
      bool cross = false;
      for (int i = 0; i < 4; ++i) cross |= (h->nbr.nb[e * 4 + i] < nc) != (e < nc);
      if (!cross) continue;
      if (e < nc) { s1[e] = next; next += 2; }
      else bslot[e] = next++;
    }
    for (int64_t e = 0; e < h->nlocal; ++e) {
      if (s1[e] >= 0) {
        lst[0].insert(lst[0].end(), {s1[e], e, 0});
        lst[1].insert(lst[1].end(), {s1[e] + 1, e, s1[e]});
      }
      if (bslot[e] >= 0) lst[2].insert(lst[2].end(), {bslot[e], e, 0});
    }
    h->nslots = (next + kLanes - 1) / kLanes * kLanes;
    for (int k = 0; k < 3; ++k) nbt[k] = nb_local;
    for (int64_t l = 0; l < h->nlocal; ++l)
      for (int i = 0; i < 4; ++i) {
        const int64_t n = h->nbr.nb[l * 4 + i];
        const size_t dst = ((l / kLanes) * 4 + i) * kLanes + l % kLanes;
        if (l >= nc && n < nc) {  // fine element, coarse neighbour: its sub-interval traces
          nbt[0][dst] = static_cast<int32_t>(s1[n]);
          nbt[1][dst] = static_cast<int32_t>(s1[n] + 1);
        } else if (l < nc && n >= nc) {  // coarse element, fine neighbour: the fine sum
          nbt[2][dst] = static_cast<int32_t>(bslot[n]);
        }
      }
  }
  const int eb = elem_bytes(h);
  const size_t q_n = static_cast<size_t>(h->ntiles) * kLanes * h->P * h->B;
  const size_t tr_n = static_cast<size_t>(h->nslots) * 4 * (trace_block(h) ? trace_block(h) : h->Bt * h->P);
  if ((rc = dalloc(h, &h->Q, q_n * eb))) { free_mesh(h); return rc; }
  if ((rc = dalloc(h, &h->traces, tr_n * eb))) { free_mesh(h); return rc; }
  if ((rc = dalloc(h, reinterpret_cast<void**>(&h->nb), nb_local.size() * sizeof(int32_t)))) { free_mesh(h); return rc; }
  if ((rc = dalloc(h, reinterpret_cast<void**>(&h->jh), jh_local.size()))) { free_mesh(h); return rc; }
  CUDA_OR_FAIL(h, cudaMemset(h->Q, 0, q_n * eb));
  CUDA_OR_FAIL(h, cudaMemset(h->traces, 0, tr_n * eb));
  // fused step kernel (YDG_FUSED=1; measured slower: the two kernels' code
  // does not fit the SM's instruction cache together): a second trace buffer, if the device
  // has room for it with 2 GB to spare
  {
    const char* fz = std::getenv("YDG_FUSED");
    size_t fr = 0, tot = 0;
    if (eb == 8 && h->nranks == 1 && kDmLanes == 8 && fz && std::atoi(fz) == 1 &&
        cudaMemGetInfo(&fr, &tot) == cudaSuccess && fr > tr_n * eb + (size_t(2) << 30) &&
        dalloc(h, &h->traces2, tr_n * eb) == YDG_OK) {
      CUDA_OR_FAIL(h, cudaMemset(h->traces2, 0, tr_n * eb));
      h->fused = true;
    }
  }
  CUDA_OR_FAIL(h, cudaMemcpy(h->nb, nb_local.data(), nb_local.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  CUDA_OR_FAIL(h, cudaMemcpy(h->jh, jh_local.data(), jh_local.size(), cudaMemcpyHostToDevice));
  if (h->lts) {
    for (int k = 0; k < 3; ++k) {
      if ((rc = dalloc(h, reinterpret_cast<void**>(&h->nb_lts[k]), nbt[k].size() * sizeof(int32_t)))) { free_mesh(h); return rc; }
      CUDA_OR_FAIL(h, cudaMemcpy(h->nb_lts[k], nbt[k].data(), nbt[k].size() * sizeof(int32_t), cudaMemcpyHostToDevice));
      h->lts_n[k] = static_cast<int64_t>(lst[k].size() / 3);
      if ((rc = dalloc(h, reinterpret_cast<void**>(&h->lts_lst[k]), std::max<size_t>(1, lst[k].size()) * sizeof(int64_t)))) { free_mesh(h); return rc; }
      if (!lst[k].empty())
        CUDA_OR_FAIL(h, cudaMemcpy(h->lts_lst[k], lst[k].data(), lst[k].size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    }
  }
  rc = eb == 8 ? upload_coeffs<double>(h, xyz, material, anelastic) : upload_coeffs<float>(h, xyz, material, anelastic);
  if (rc) { free_mesh(h); return rc; }
  if (h->nranks > 1) {
    rc = h->halo.bind(h->traces, h->Bt, h->P, trace_block(h), h->lanes, eb, owned_slots, &h->err);
    if (rc) { free_mesh(h); return fail(h, rc, h->err); }
  }
  // staging buffer for DOF transfers (bounded)
  h->staging_bytes = std::min<size_t>(q_n * eb, size_t(256) << 20);
  if ((rc = dalloc(h, &h->staging, h->staging_bytes))) { free_mesh(h); return rc; }
  // grids: resident CTAs per SM x SMs
  int sms = 0, occ_l = 0, occ_n = 0;
  CUDA_OR_FAIL(h, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->dev));
  occ_l = eb == 8 ? kDmCtasPerSm : 1;  // fp64: 12 warps per SM in kDmCtasPerSm work groups
  // fp64 flux kernel: 3-warp groups (8-element halves); four single-group CTAs per SM, or
  // one CTA of kFluxGroups groups
  occ_n = eb == 8 ? (kFluxGroups > 1 ? kFluxGroups : 4) : 1;
  h->grid_local = sms * occ_l;
  h->grid_neigh = sms * occ_n;
  // YDG_GRID_LOCAL / YDG_GRID_NEIGH (tests): other persistent grid sizes (virtual CTAs), so
  // that a race between work groups shows up as a bitwise difference of the results
  if (const char* gl = std::getenv("YDG_GRID_LOCAL")) h->grid_local = std::max(1, std::atoi(gl));
  if (const char* gn = std::getenv("YDG_GRID_NEIGH")) h->grid_neigh = std::max(1, std::atoi(gn));
  h->have_mesh = true;
  return YDG_OK;
}

static int xfer_dofs(ydg_solver* h, int64_t first, int64_t count, const void* src_host, void* dst_host,
                     const void* src_dev, void* dst_dev, cudaStream_t s, bool upload) {
  int rc = check(h);
  if (rc) return rc;
  if (!h->have_mesh) return fail(h, YDG_ERR_STATE, "upload the mesh first");
  if (count < 0 || first < h->first || first + count > h->first + h->nlocal)
    return fail(h, YDG_ERR_ARG, "element range not owned by this rank");
  // host transfers are blocking: wait for steps enqueued on any stream
  if (!src_dev && !dst_dev) CUDA_OR_FAIL(h, cudaDeviceSynchronize());
  const int eb = elem_bytes(h);
  const int64_t per = static_cast<int64_t>(h->P) * h->B;
  const bool dev_side = src_dev || dst_dev;
  if (h->generic) {  // canonical layout on the device: plain copies
    char* q = static_cast<char*>(h->Q) + (first - h->first) * per * eb;
    const size_t bytes = static_cast<size_t>(count) * per * eb;
    if (upload)
      CUDA_OR_FAIL(h, cudaMemcpyAsync(q, src_dev ? src_dev : src_host, bytes, cudaMemcpyDefault, s));
    else
      CUDA_OR_FAIL(h, cudaMemcpyAsync(dst_dev ? dst_dev : dst_host, q, bytes, cudaMemcpyDefault, s));
    if (!dev_side) CUDA_OR_FAIL(h, cudaStreamSynchronize(s));
    return YDG_OK;
  }
  const int64_t chunk = dev_side ? count : std::max<int64_t>(1, static_cast<int64_t>(h->staging_bytes) / (per * eb));
  for (int64_t c0 = 0; c0 < count; c0 += chunk) {
    const int64_t n = std::min(chunk, count - c0);
    const int64_t lfirst = first - h->first + c0;
    void* buf = h->staging;
    if (upload) {
      if (dev_side) {
        buf = const_cast<void*>(static_cast<const void*>(static_cast<const char*>(src_dev) + c0 * per * eb));
      } else {
        CUDA_OR_FAIL(h, cudaMemcpyAsync(buf, static_cast<const char*>(src_host) + c0 * per * eb, n * per * eb,
                                        cudaMemcpyHostToDevice, s));
      }
      cudaError_t e = eb == 8 ? launch_to_tiled<double>(h->P, h->B, h->lanes, static_cast<const double*>(buf), static_cast<double*>(h->Q), lfirst, n, h->slot_of, s)
                              : launch_to_tiled<float>(h->P, h->B, h->lanes, static_cast<const float*>(buf), static_cast<float*>(h->Q), lfirst, n, h->slot_of, s);
      CUDA_OR_FAIL(h, e);
      if (!dev_side) CUDA_OR_FAIL(h, cudaStreamSynchronize(s));
    } else {
      if (dev_side) buf = static_cast<char*>(dst_dev) + c0 * per * eb;
      cudaError_t e = eb == 8 ? launch_to_canonical<double>(h->P, h->B, h->lanes, static_cast<const double*>(h->Q), static_cast<double*>(buf), lfirst, n, h->slot_of, s)
                              : launch_to_canonical<float>(h->P, h->B, h->lanes, static_cast<const float*>(h->Q), static_cast<float*>(buf), lfirst, n, h->slot_of, s);
      CUDA_OR_FAIL(h, e);
      if (!dev_side) {
        CUDA_OR_FAIL(h, cudaMemcpyAsync(static_cast<char*>(dst_host) + c0 * per * eb, buf, n * per * eb,
                                        cudaMemcpyDeviceToHost, s));
        CUDA_OR_FAIL(h, cudaStreamSynchronize(s));
      }
    }
  }
  return YDG_OK;
}

int ydg_upload_dofs(ydg_solver* h, int64_t first, int64_t count, const void* Q) {
  if (!Q) return h ? fail(h, YDG_ERR_ARG, "null Q") : YDG_ERR_ARG;
  return xfer_dofs(h, first, count, Q, nullptr, nullptr, nullptr, h ? h->stream : nullptr, true);
}
int ydg_download_dofs(ydg_solver* h, int64_t first, int64_t count, void* Q_out) {
  if (!Q_out) return h ? fail(h, YDG_ERR_ARG, "null Q_out") : YDG_ERR_ARG;
  return xfer_dofs(h, first, count, nullptr, Q_out, nullptr, nullptr, h ? h->stream : nullptr, false);
}
int ydg_upload_dofs_device(ydg_solver* h, int64_t first, int64_t count, const void* Q_dev, void* s) {
  if (!Q_dev) return h ? fail(h, YDG_ERR_ARG, "null Q_dev") : YDG_ERR_ARG;
  return xfer_dofs(h, first, count, nullptr, nullptr, Q_dev, nullptr, h ? pick_stream(h, s) : nullptr, true);
}
int ydg_download_dofs_device(ydg_solver* h, int64_t first, int64_t count, void* Q_dev, void* s) {
  if (!Q_dev) return h ? fail(h, YDG_ERR_ARG, "null Q_dev") : YDG_ERR_ARG;
  return xfer_dofs(h, first, count, nullptr, nullptr, nullptr, Q_dev, h ? pick_stream(h, s) : nullptr, false);
}

int ydg_step(ydg_solver* h, double dt, int nsteps, void* cuda_stream) {
  int rc = check(h);
  if (rc) return rc;
  if (!h->have_mesh) return fail(h, YDG_ERR_STATE, "upload the mesh first");
  if (!(dt > 0) || !std::isfinite(dt) || nsteps < 0) return fail(h, YDG_ERR_ARG, "bad dt or nsteps");
  cudaStream_t s = pick_stream(h, cuda_stream);
  if (h->generic) return generic_step(h, dt, nsteps, s);
  return h->prec == 8 ? do_step<double>(h, dt, nsteps, s) : do_step<float>(h, dt, nsteps, s);
}

int ydg_step_graph(ydg_solver* h, double dt, int nsteps, void* cuda_stream) {
  int rc = check(h);
  if (rc) return rc;
  if (!h->have_mesh) return fail(h, YDG_ERR_STATE, "upload the mesh first");
  if (!(dt > 0) || !std::isfinite(dt) || nsteps < 0) return fail(h, YDG_ERR_ARG, "bad dt or nsteps");
  if (h->nranks > 1) return fail(h, YDG_ERR_UNSUPPORTED, "ydg_step_graph runs on one rank (the halo has host barriers)");
  if (h->profiling) return fail(h, YDG_ERR_STATE, "disable ydg_profile before ydg_step_graph");
  if (nsteps == 0) return YDG_OK;
  cudaStream_t s = pick_stream(h, cuda_stream);
  if (!h->gexec || h->g_dt != dt || h->g_n != nsteps) {
    if (h->gexec) cudaGraphExecDestroy(h->gexec);
    h->gexec = nullptr;
    if (!h->cap_stream) CUDA_OR_FAIL(h, cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
    CUDA_OR_FAIL(h, cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeRelaxed));
    rc = h->generic ? generic_step(h, dt, nsteps, h->cap_stream)
                    : (h->prec == 8 ? do_step<double>(h, dt, nsteps, h->cap_stream)
                                    : do_step<float>(h, dt, nsteps, h->cap_stream));
    cudaGraph_t g = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(h->cap_stream, &g);
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    CUDA_OR_FAIL(h, ec);
    const cudaError_t ei = cudaGraphInstantiate(&h->gexec, g, 0);
    cudaGraphDestroy(g);
    CUDA_OR_FAIL(h, ei);
    h->g_dt = dt;
    h->g_n = nsteps;
  }
  CUDA_OR_FAIL(h, cudaGraphLaunch(h->gexec, s));
  return YDG_OK;
}

int ydg_set_clusters(ydg_solver* h, const int8_t* cluster, int64_t n) {
  int rc = check(h);
  if (rc) return rc;
  if (h->have_mesh) return fail(h, YDG_ERR_STATE, "ydg_set_clusters must precede ydg_upload_mesh");
  if (!cluster || n < 0) return fail(h, YDG_ERR_ARG, "null cluster array");
  for (int64_t e = 0; e < n; ++e)
    if (cluster[e] != 0 && cluster[e] != 1) return fail(h, YDG_ERR_ARG, "cluster ids must be 0 (dt) or 1 (2 dt)");
  h->cluster_ext.assign(cluster, cluster + n);
  return YDG_OK;
}

int ydg_step_lts(ydg_solver* h, double dt, int ncycles, void* cuda_stream) {
  int rc = check(h);
  if (rc) return rc;
  if (!h->have_mesh) return fail(h, YDG_ERR_STATE, "upload the mesh first");
  if (!h->lts) return fail(h, YDG_ERR_STATE, "no clusters: call ydg_set_clusters before ydg_upload_mesh");
  if (!(dt > 0) || !std::isfinite(dt) || ncycles < 0) return fail(h, YDG_ERR_ARG, "bad dt or ncycles");
  cudaStream_t s = pick_stream(h, cuda_stream);
  StepParams<double> base{};
  base.Q = static_cast<double*>(h->Q);
  base.traces = static_cast<double*>(h->traces);
  base.star = static_cast<const double*>(h->star);
  base.aplus = static_cast<const double*>(h->aplus);
  base.jh = h->jh;
  auto with_dt = [&](double tau) {
    StepParams<double> p = base;
    p.dt = tau;
    for (int d = 0; d < h->N; ++d) {
      p.scal[d] = tau / (d + 1);
      p.scal[h->N + d] = tau / (d + 2);
    }
    return p;
  };
  const int64_t ntc = h->lts_nc / h->lanes, ntf = h->ntiles - ntc;
  const int TS = trace_block(h);
  auto local = [&](StepParams<double> p, int64_t t0, int64_t nt, int tr_only) -> int {
    if (nt <= 0) return YDG_OK;
    p.nb = h->nb;
    p.tile0 = t0;
    p.ntiles = nt;
    p.tr_only = tr_only;
    CUDA_OR_FAIL(h, timed(h, 0, s, [&] { return launch_local<double>(h->N, p, static_cast<int>(std::min<int64_t>(h->grid_local, nt)), s); }));
    return YDG_OK;
  };
  auto flux = [&](int table, int64_t t0, int64_t nt) -> int {
    if (nt <= 0) return YDG_OK;
    StepParams<double> p = base;
    p.nb = h->nb_lts[table];
    p.tile0 = t0;
    p.ntiles = nt;
    CUDA_OR_FAIL(h, timed(h, 1, s, [&] { return launch_neigh<double>(h->N, p, static_cast<int>(std::min<int64_t>(h->grid_neigh, nt * (h->lanes / 8))), s); }));
    return YDG_OK;
  };
  auto combine = [&](int k, int mode) -> int {
    CUDA_OR_FAIL(h, launch_trace_combine(static_cast<double*>(h->traces), h->lts_lst[k], h->lts_n[k], TS, h->lanes, mode, s));
    return YDG_OK;
  };
  const StepParams<double> p1 = with_dt(dt), p2 = with_dt(2 * dt);
  for (int c = 0; c < ncycles; ++c) {
    // coarse elements next to fine ones: traces of I[0, dt] -> S1 (before their update)
    if ((rc = local(p1, 0, h->lts_ncb_tiles, 1)) || (rc = combine(0, 0))) return rc;
    // coarse: traces of I[0, 2 dt], volume update; S2 = I[0, 2dt] - I[0, dt] traces
    if ((rc = local(p2, 0, ntc, 0)) || (rc = combine(1, 1))) return rc;
    // fine substep 1: local (dt), B = own traces, flux with the coarse S1
    if ((rc = local(p1, ntc, ntf, 0)) || (rc = combine(2, 0)) || (rc = flux(0, ntc, ntf))) return rc;
    // fine substep 2: local (dt) from the updated Q, B += own traces, flux with S2
    if ((rc = local(p1, ntc, ntf, 0)) || (rc = combine(2, 2)) || (rc = flux(1, ntc, ntf))) return rc;
    // coarse flux over 2 dt: coarse neighbours' full traces, fine neighbours' B
    if ((rc = flux(2, 0, ntc))) return rc;
  }
  return YDG_OK;
}

int ydg_synchronize(ydg_solver* h) {
  int rc = check(h);
  if (rc) return rc;
  CUDA_OR_FAIL(h, cudaStreamSynchronize(h->stream));
  CUDA_OR_FAIL(h, cudaDeviceSynchronize());
  return YDG_OK;
}

int ydg_get_neighbours(ydg_solver* h, int64_t first, int64_t count, int64_t* nb, int8_t* j, int8_t* hr) {
  int rc = check(h);
  if (rc) return rc;
  if (!h->have_mesh) return fail(h, YDG_ERR_STATE, "upload the mesh first");
  if (!nb || !j || !hr || count < 0 || first < 0 || first + count > h->ne)
    return fail(h, YDG_ERR_ARG, "bad neighbour query");
  const Neighbours& t = h->nbr_ext.nb.empty() ? h->nbr : h->nbr_ext;
  std::memcpy(nb, t.nb.data() + first * 4, count * 4 * sizeof(int64_t));
  std::memcpy(j, t.j.data() + first * 4, count * 4);
  std::memcpy(hr, t.h.data() + first * 4, count * 4);
  return YDG_OK;
}

int ydg_halo_plan(int64_t ne, const int64_t* vid, int rank, int nranks, int64_t* counts,
                  int32_t* peers, int64_t* recv_cnt, int64_t* send_cnt, int64_t* ghost_of,
                  int64_t* send_elem, int8_t* send_face, int64_t* recv_elem, int8_t* recv_face) {
  if (ne <= 0 || !vid || !counts || nranks < 1 || rank < 0 || rank >= nranks) return YDG_ERR_ARG;
  Neighbours nbr;
  std::string err;
  if (!match_faces(ne, vid, &nbr, &err)) {
    g_last_error = err;
    return YDG_ERR_MESH;
  }
  HaloPlan plan;
  if (!plan_halo(nbr, ne, rank, nranks, &plan, &err)) {
    g_last_error = err;
    return YDG_ERR_MESH;
  }
  counts[0] = static_cast<int64_t>(plan.peers.size());
  counts[1] = static_cast<int64_t>(plan.ghost_of.size());
  counts[2] = static_cast<int64_t>(plan.send_slots.size());
  const int64_t first = ne * rank / nranks;
  if (peers && recv_cnt && send_cnt)
    for (size_t k = 0; k < plan.peers.size(); ++k) {
      peers[k] = plan.peers[k];
      recv_cnt[k] = plan.recv_cnt[k];
      send_cnt[k] = plan.send_cnt[k];
    }
  if (ghost_of) std::copy(plan.ghost_of.begin(), plan.ghost_of.end(), ghost_of);
  for (size_t k = 0; k < plan.send_slots.size(); ++k) {
    if (send_elem) send_elem[k] = first + plan.send_slots[k];
    if (send_face) send_face[k] = plan.send_face[k];
  }
  for (size_t k = 0; k < plan.recv_ghost.size(); ++k) {
    if (recv_elem) recv_elem[k] = plan.ghost_of[plan.recv_ghost[k]];
    if (recv_face) recv_face[k] = plan.recv_face[k];
  }
  return YDG_OK;
}

int ydg_profile(ydg_solver* h, int enable) {
  int rc = check(h);
  if (rc) return rc;
  if ((rc = drain_profile(h))) return rc;
  h->profiling = enable != 0;
  h->prof_ms[0] = h->prof_ms[1] = h->prof_ms[2] = 0;
  h->prof_launches = 0;
  return YDG_OK;
}

int ydg_query(ydg_solver* h, int what, double* v) {
  if (!h || !v) return YDG_ERR_ARG;
  if ((what >= YDG_Q_PROF_LOCAL_MS && what <= YDG_Q_PROF_LAUNCHES) || what == YDG_Q_PROF_FUSED_MS) {
    int rc = check(h);
    if (rc) return rc;
    if ((rc = drain_profile(h))) return rc;
  }
  switch (what) {
    case YDG_Q_PROF_LOCAL_MS: *v = h->prof_ms[0]; break;
    case YDG_Q_PROF_NEIGH_MS: *v = h->prof_ms[1]; break;
    case YDG_Q_PROF_LAUNCHES: *v = static_cast<double>(h->prof_launches); break;
    case YDG_Q_PROF_FUSED_MS: *v = h->prof_ms[2]; break;
    case YDG_Q_FUSED: *v = h->fused ? 1.0 : 0.0; break;
    case YDG_Q_FUSED_BYTES: *v = h->prec == 8 && !h->generic ? alg_bytes_fused(h) : 0.0; break;
    case YDG_Q_SIMULATIONS: *v = static_cast<double>(h->sims); break;
    case YDG_Q_GUARD_VIOLATIONS: *v = h->guard ? static_cast<double>(guard_violations(h)) : -1.0; break;
    case YDG_Q_MAX_ABS_Q: {
      int rc = check(h);
      if (rc) return rc;
      if (!h->have_mesh) return fail(h, YDG_ERR_STATE, "no mesh");
      *v = max_abs_q(h);
      break;
    }
    case YDG_Q_TILE_ELEMENTS: *v = static_cast<double>(h->prec == 8 ? kDmLanes : kLanes); break;
    case YDG_Q_N_ELEMENTS: *v = static_cast<double>(h->ne); break;
    case YDG_Q_FIRST_LOCAL: *v = static_cast<double>(h->first); break;
    case YDG_Q_N_LOCAL: *v = static_cast<double>(h->nlocal); break;
    // canonical formulation of P:1312-1342 (local and neighbour flux with their own lifts,
    // DESIGN.md R22); the fp64 kernels execute fewer (one lift per face) -- not counted
    case YDG_Q_NZ_FLOPS: *v = h->P == 27 ? nz_flops_visco(h->N) : nz_flops_elastic(h->N, false); break;
    case YDG_Q_ALG_BYTES: *v = alg_bytes_local(h) + alg_bytes_neigh(h); break;
    case YDG_Q_B: *v = h->B; break;
    case YDG_Q_BTILDE: *v = h->Bt; break;
    case YDG_Q_DEVICE_BYTES: *v = static_cast<double>(h->device_bytes); break;
    case YDG_Q_LAUNCHES_PER_STEP: *v = h->nranks > 1 ? 5 : 2; break;
    case YDG_Q_LOCAL_BYTES: *v = alg_bytes_local(h); break;
    case YDG_Q_NEIGH_BYTES: *v = alg_bytes_neigh(h); break;
    case YDG_Q_KERNEL_PATH: *v = h->generic ? (h->visco_tc ? 2 : 3) : (h->prec == 8 ? 0 : 1); break;
    // tiled elastic kernels (fp64, fp32): the local kernel runs CK, time integral, volume,
    // traces; both flux terms are in the flux kernel.  Generic CSR path: the local flux is
    // in the local kernel.
    case YDG_Q_LOCAL_FLOPS: *v = h->P == 27 ? nz_flops_visco_local(h->N) : nz_flops_local(h->N, shared_lift(h)); break;
    case YDG_Q_NEIGH_FLOPS:
      *v = h->P == 27 ? nz_flops_visco(h->N) - nz_flops_visco_local(h->N)
                      : nz_flops_elastic(h->N, false) - nz_flops_local(h->N, shared_lift(h));
      break;
    case YDG_Q_NEIGH_FLOPS_EXEC:  // the tiled flux kernels lift local + neighbour flux once per face
      *v = h->P == 27 ? nz_flops_visco(h->N) - nz_flops_visco_local(h->N)
                      : nz_flops_elastic(h->N, shared_lift(h)) - nz_flops_local(h->N, shared_lift(h));
      break;
    default: return fail(h, YDG_ERR_ARG, "unknown query");
  }
  return YDG_OK;
}

const char* ydg_error_string(const ydg_solver* h) { return h ? h->err.c_str() : "null handle"; }

void ydg_destroy(ydg_solver* h) {
  if (!h) return;
  cudaSetDevice(h->dev);
  if (h->stream) cudaStreamSynchronize(h->stream);
  drain_profile(h);
  free_mesh(h);
  for (void* p : h->csr) cudaFree(p);
  h->halo.destroy();
  if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

}  // extern "C"
