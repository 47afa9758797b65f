// FP64 tensor-core (DMMA m8n8k4) kernels of the ADER-DG update (sm_100a, fp64).
//
// Data of a 32-element tile live in shared memory as [row][col] with col = p*32 + e
// (quantity-major), rows swizzled (col ^ 8*(row & 1)) so that the 4-row x 8-column DMMA
// B-fragment loads take the minimum two wavefronts and per-thread column accesses stay
// conflict-free.  Warp p owns the four 8-column tiles of quantity p: every B operand it
// feeds to a DMMA is warp-private; only the per-element quantity mixing (star matrices
// A*, flux solvers A+-) reads other warps' columns.  Global matrices are the DMMA A
// operands (generated 8x4 tiles, zero tiles skipped: gen/dmma.py).
#pragma once
#include "kernels.cuh"

namespace ydg {
namespace dm {

constexpr int kP = 9;
constexpr int kL = 32;
constexpr int kRS = kP * kL;   // 288 columns per row
constexpr int kXB = 40;        // padded row of the warp-private X buffer (2 wavefronts / B load)

enum Src { SRC_Q, SRC_S, SRC_I };

__device__ __forceinline__ int swz(int row, int col) { return row * kRS + (col ^ ((row & 1) << 3)); }

struct Ctx {
  int lane, p;
  double* S;          // [SROWS][288]  D^d, d >= 1
  double* I;          // [IROWS][288]  time integral rows < IROWS
  double* xb;         // warp-private [3][4][kXB]
  const double* Qt;   // Q of this tile in global memory: [B][9][32]
  const double* frags;
  double a[9];        // star matrices, row p: a[3c + j] = A*^c[p][q_j]
  int q0, q1, q2;     // star columns of row p
  double dt;
  const double* scal;  // kernel-parameter space: dt/(d+1) at [d], dt/(d+2) at [N + d]
  int N;
};

template <int N>
struct DG;
template <int N>
__device__ const double* frag_table();

__device__ __forceinline__ double afrag(const Ctx& x, int tid) { return __ldg(x.frags + tid * kL + x.lane); }

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}
__device__ __forceinline__ void dmma4(double (&acc)[4][2], double a, const double (&bf)[4]) {
#pragma unroll
  for (int ct = 0; ct < 4; ++ct) dmma(acc[ct], a, bf[ct]);
}

template <int MT>
__device__ __forceinline__ void zero_acc(double (&acc)[MT][4][2]) {
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[m][c][0] = acc[m][c][1] = 0.0;
}

template <Src SRC, int B>
__device__ __forceinline__ double load_data(const Ctx& x, int row, int col) {
  // Q^n of the tile is staged in shared memory at the rows of I (rows >= IROWS continue
  // into S) for the first CK step
  if constexpr (SRC == SRC_Q) return row < B ? x.I[swz(row, col)] : 0.0;
  else if constexpr (SRC == SRC_S) return x.S[swz(row, col)];
  else return x.I[swz(row, col)];
}

// X^c = D A*^cT for rows l0..l0+3 of the thread's own column (element lane, quantity p),
// staged in the warp-private buffer [c][r][kXB]; xb_b then reads one c's B fragments
// for the warp's four column tiles.  The caller ends the k-step with __syncwarp().
template <Src SRC, int B>
__device__ __forceinline__ void xchunk(Ctx& x, int l0) {
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const double d0 = load_data<SRC, B>(x, l0 + r, x.q0 * kL + x.lane);
    const double d1 = load_data<SRC, B>(x, l0 + r, x.q1 * kL + x.lane);
    const double d2 = load_data<SRC, B>(x, l0 + r, x.q2 * kL + x.lane);
#pragma unroll
    for (int c = 0; c < 3; ++c)
      x.xb[(c * 4 + r) * kXB + x.lane] = fma(x.a[3 * c + 2], d2, fma(x.a[3 * c + 1], d1, x.a[3 * c] * d0));
  }
  __syncwarp();
}
__device__ __forceinline__ void xb_b(const Ctx& x, int c, double (&bf)[4]) {
#pragma unroll
  for (int ct = 0; ct < 4; ++ct) bf[ct] = x.xb[(c * 4 + (x.lane & 3)) * kXB + 8 * ct + (x.lane >> 2)];
}

// B fragments of the time integral (own quantity p): rows < IROWS from shared memory
// (ismem_b); the remaining rows are dt * Q (only D^0 contributes to them), read from global
// memory (gq_b) at the start of each trace so that their latency overlaps the DMMAs.
__device__ __forceinline__ void ismem_b(const Ctx& x, int l0, double (&bf)[4]) {
  const int row = l0 + (x.lane & 3);
#pragma unroll
  for (int ct = 0; ct < 4; ++ct) bf[ct] = x.I[swz(row, x.p * kL + 8 * ct + (x.lane >> 2))];
}
template <int B>
__device__ __forceinline__ void gq_b(const Ctx& x, int l0, double (&bf)[4]) {
  const int row = l0 + (x.lane & 3);
#pragma unroll
  for (int ct = 0; ct < 4; ++ct)
    bf[ct] = row < B ? x.dt * x.Qt[row * kRS + x.p * kL + 8 * ct + (x.lane >> 2)] : 0.0;
}

__device__ __forceinline__ void smem_b(const Ctx& x, const double* Y, int l0, double (&bf)[4]) {
  const int row = l0 + (x.lane & 3);
#pragma unroll
  for (int ct = 0; ct < 4; ++ct) bf[ct] = Y[swz(row, x.p * kL + 8 * ct + (x.lane >> 2))];
}

// Write D^{d+1} = dt/(d+1) acc into S and accumulate the time integral;
// at d = 0 the integral starts from dt * Q.
template <int MT, int FIRST, int B>
__device__ __forceinline__ void ck_writeback(Ctx& x, const double (&acc)[MT][4][2], int d) {
  const double sc = x.scal[d], ic = x.scal[x.N + d];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) {
      const int row = 8 * mt + (x.lane >> 2);
      const int col = x.p * kL + 8 * ct + 2 * (x.lane & 3);
      const int s = swz(row, col);
      const double v0 = sc * acc[mt][ct][0], v1 = sc * acc[mt][ct][1];
      *reinterpret_cast<double2*>(x.S + s) = make_double2(v0, v1);
      double2 i2;
      if (FIRST) {
        const double2 q = row < B ? *reinterpret_cast<const double2*>(x.I + s) : make_double2(0.0, 0.0);
        i2 = make_double2(fma(ic, v0, x.dt * q.x), fma(ic, v1, x.dt * q.y));
      } else {
        i2 = *reinterpret_cast<const double2*>(x.I + s);
        i2.x = fma(ic, v0, i2.x);
        i2.y = fma(ic, v1, i2.y);
      }
      *reinterpret_cast<double2*>(x.I + s) = i2;
    }
}

// Q += acc, direct read-modify-write of the C fragments in global memory.
template <int MT, int B>
__device__ __forceinline__ void add_q(const Ctx& x, double* Qt, const double (&acc)[MT][4][2]) {
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) {
      if (8 * mt + (x.lane >> 2) >= B) continue;
      double2* q = reinterpret_cast<double2*>(Qt + (8 * mt + (x.lane >> 2)) * kRS + x.p * kL + 8 * ct +
                                              2 * (x.lane & 3));
      double2 v = *q;
      v.x += acc[mt][ct][0];
      v.y += acc[mt][ct][1];
      *q = v;
    }
}

// Q += acc (C fragments of 8-row tiles, rows < B): the fragments go to a shared staging
// region [B][288] (stage_acc, then a barrier), then every thread updates Q with coalesced
// 16-byte read-modify-writes (update_q) -- no accumulator is live while Q is loaded.
template <int MT, int B>
__device__ __forceinline__ void stage_acc(const Ctx& x, double* st, const double (&acc)[MT][4][2]) {
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) {
      const int row = 8 * mt + (x.lane >> 2);
      if (row >= B) continue;
      *reinterpret_cast<double2*>(st + swz(row, x.p * kL + 8 * ct + 2 * (x.lane & 3))) =
          make_double2(acc[mt][ct][0], acc[mt][ct][1]);
    }
}
#ifndef YDG_QSTAGE
#define YDG_QSTAGE 0
#endif
template <int B>
__device__ __forceinline__ void update_q(double* Qt, const double* st) {
  constexpr int kPairs = B * kRS / 2;
#pragma unroll 4
  for (int c = threadIdx.x; c < kPairs; c += kP * kL) {
    const int row = c / (kRS / 2), cc = 2 * (c % (kRS / 2));
    double2* q = reinterpret_cast<double2*>(Qt + row * kRS + cc);
    const double2 a = *reinterpret_cast<const double2*>(st + swz(row, cc));
    double2 v = *q;
    v.x += a.x;
    v.y += a.y;
    *q = v;
  }
}

// Store the trace C fragments (rows < Bt) to global memory [tile][face][m][q][32].
template <int MT, int Bt>
__device__ __forceinline__ void store_trace_global(const Ctx& x, double* gtr, const double (&acc)[MT][4][2]) {
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) {
      const int row = 8 * mt + (x.lane >> 2);
      const int col = x.p * kL + 8 * ct + 2 * (x.lane & 3);
      if (row < Bt) *reinterpret_cast<double2*>(gtr + row * kRS + col) = make_double2(acc[mt][ct][0], acc[mt][ct][1]);
    }
}

// Y = Z A^T per element (thread = element lane, quantity p), in place in the staging region
// (all columns of Z are read before the barrier, then each thread writes its own column).
template <int Bt>
__device__ __forceinline__ void mix_inplace(const Ctx& x, double* Z, const double* flux, int64_t tile,
                                            int F) {
  double arow[kP];
  const double* A = flux + ((tile * 4 + F) * kP + x.p) * kP * kL + x.lane;
#pragma unroll
  for (int q = 0; q < kP; ++q) arow[q] = A[q * kL];
  double y[Bt];
#pragma unroll
  for (int m = 0; m < Bt; ++m) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < kP; ++q) s = fma(Z[swz(m, q * kL + x.lane)], arow[q], s);
    y[m] = s;
  }
  __syncthreads();
#pragma unroll
  for (int m = 0; m < Bt; ++m) Z[swz(m, x.p * kL + x.lane)] = y[m];
}

// Y = T A^T with T read from the tile's traces in global memory ([m][q][32] rows of face
// F), written to the own column of a shared staging region; no barrier needed since the
// lift that consumes Y reads only the warp's own columns.
template <int Bt>
__device__ __forceinline__ void mix_from_global(const Ctx& x, double* Y, const double* gT,
                                                const double* flux, int64_t tile, int F) {
  double arow[kP];
  const double* A = flux + ((tile * 4 + F) * kP + x.p) * kP * kL + x.lane;
#pragma unroll
  for (int q = 0; q < kP; ++q) arow[q] = A[q * kL];
#pragma unroll 3
  for (int m = 0; m < Bt; ++m) {
    const double* row = gT + m * kRS + x.lane;
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < kP; ++q) s = fma(row[q * kL], arow[q], s);
    Y[swz(m, x.p * kL + x.lane)] = s;
  }
}

template <int N>
struct Layout {
  using G = DG<N>;
  static constexpr int XB = 9 * 3 * 4 * kXB;  // doubles
  // local kernel: [I][S][xb]; the face staging region (TROWS rows) reuses S
  // [I][S][xb]; Q^n of the tile is staged over I and S for the first CK step
  static constexpr int LOCAL = (G::IROWS + G::SROWS > G::B ? G::IROWS + G::SROWS : G::B) * kRS + XB;
  // Z, T, mbarrier (the Q-update staging [B][288] reuses Z and T)
  static constexpr int NEIGH = (2 * G::TROWS + 2 * G::Bt > G::B ? 2 * G::TROWS + 2 * G::Bt : G::B) * kRS + 2;
};

// ---- asynchronous copy helpers (TMA bulk copy + mbarrier, Ampere-style cp.async)
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// CK + time integral, face traces R^iT I (stored for the flux kernel) and
// the volume term for 32-element tiles.
template <int N>
__global__ void __launch_bounds__(kP * kL, 1) dm_local(const __grid_constant__ StepParams<double> prm) {
  using G = DG<N>;
  constexpr int B = G::B, Bt = G::Bt;
  extern __shared__ __align__(16) double smem[];
  Ctx x;
  x.lane = threadIdx.x & 31;
  x.p = threadIdx.x >> 5;
  x.I = smem;
  x.S = smem + G::IROWS * kRS;
  x.xb = smem + (G::IROWS + G::SROWS > B ? G::IROWS + G::SROWS : B) * kRS + x.p * (3 * 4 * kXB);
  x.frags = frag_table<N>();
  x.dt = prm.dt;
  x.scal = prm.scal;
  x.N = N;
  // 3-column pattern of star-matrix row p (setup.cpp star_cols), packed 5 bits per column
  {
    constexpr unsigned long long packed[9] = {6 | 7 << 5 | 8 << 10, 6 | 7 << 5 | 8 << 10, 6 | 7 << 5 | 8 << 10,
                                              6 | 7 << 5 | 7 << 10, 7 | 8 << 5 | 8 << 10, 6 | 8 << 5 | 8 << 10,
                                              0 | 3 << 5 | 5 << 10, 3 | 1 << 5 | 4 << 10, 5 | 4 << 5 | 2 << 10};
    unsigned long long w = 0;
#pragma unroll
    for (int i = 0; i < 9; ++i) w = (x.p == i) ? packed[i] : w;
    x.q0 = static_cast<int>(w & 31);
    x.q1 = static_cast<int>((w >> 5) & 31);
    x.q2 = static_cast<int>((w >> 10) & 31);
  }
  for (int64_t it = blockIdx.x; it < prm.ntiles; it += gridDim.x) {
    const int64_t tile = prm.tile0 + it;
    double* Qt = prm.Q + tile * B * kRS;
    if (threadIdx.x == 0 && it + gridDim.x < prm.ntiles) {  // next tile of this CTA -> L2
      const int64_t nt = tile + gridDim.x;
      prefetch_l2(prm.Q + nt * B * kRS, B * kRS * sizeof(double));
      prefetch_l2(prm.star + nt * 3 * kP * 3 * kL, 3 * kP * 3 * kL * sizeof(double));
    }
    x.Qt = Qt;
    {  // stage Q^n of the tile in shared memory (rows of I, continuing into S): 16-byte
       // cp.async chunks, all in flight at once
      constexpr int kChunks = B * kRS / 2;
      for (int c = threadIdx.x; c < kChunks; c += blockDim.x) {
        const int row = c / (kRS / 2), cc = 2 * (c % (kRS / 2));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(x.I + swz(row, cc))),
                     "l"(Qt + row * kRS + cc)
                     : "memory");
      }
    }
    const double* st = prm.star + (tile * 3 * kP) * 3 * kL + x.lane;
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int j = 0; j < 3; ++j) x.a[3 * c + j] = st[((c * kP + x.p) * 3 + j) * kL];
    cp_async_wait_all();
    __syncthreads();
    G::ck(x);  // ends with a barrier: the time integral is complete
    // traces T_F = R^FT I of the four faces -> global memory; they read Q^n (rows >=
    // IROWS of I), so they precede the update of Q
    double* gtr = prm.traces + tile * 4 * Bt * kRS;
#pragma unroll
    for (int F = 0; F < 4; ++F) {
      double tacc[G::TROWS / 8][4][2];
      zero_acc(tacc);
      if (F == 0) G::template trace<0>(x, tacc);
      else if (F == 1) G::template trace<1>(x, tacc);
      else if (F == 2) G::template trace<2>(x, tacc);
      else G::template trace<3>(x, tacc);
      store_trace_global<G::TROWS / 8, Bt>(x, gtr + F * Bt * kRS, tacc);
    }
    {
      double acc[G::QMT][4][2];
      zero_acc(acc);
      G::volume(x, acc);
#if YDG_QSTAGE
      __syncthreads();  // I, S and the X buffers are dead: stage the update over them
      stage_acc<G::QMT, B>(x, smem, acc);
    }
    __syncthreads();
    update_q<B>(Qt, smem);
#else
      add_q<G::QMT, B>(x, Qt, acc);
    }
#endif
    __syncthreads();  // before the next tile overwrites the shared regions
  }
}

// Flux kernel: local and neighbour flux with one lift per face:
//   Q += sum_i R^i ( T_i A+_i^T + (f^h_i T^nb_(j_i)) A-_i^T ).
// Two passes of two faces.  Per pass all loads are issued at once: one TMA bulk copy of the
// tile's own traces of both faces (contiguous in the [tile][face][m][q][32] layout) and
// per-thread cp.async gathers of the neighbour traces into the own column of the staging
// region Z; then f^h rotates Z in place, thread (e,p) mixes T with A+ and Z with A-, writes
// Y into Z after a barrier, and the warp lifts its own columns of Y with DMMAs.
template <int N>
__global__ void __launch_bounds__(kP * kL, 1) dm_neigh(const __grid_constant__ StepParams<double> prm) {
  using G = DG<N>;
  constexpr int B = G::B, Bt = G::Bt, TR = G::TROWS;
  extern __shared__ __align__(128) double smem[];
  double* Zs = smem;                     // [2][TR][288] swizzled (neighbour traces, then Y)
  double* Ts = smem + 2 * TR * kRS;      // [2][Bt][288] own traces (TMA copy, unswizzled)
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(Ts + 2 * Bt * kRS);
  Ctx x;
  x.lane = threadIdx.x & 31;
  x.p = threadIdx.x >> 5;
  x.frags = frag_table<N>();
  const int col = x.p * kL + x.lane;
  for (int i = threadIdx.x; i < 2 * (TR - Bt) * kRS; i += blockDim.x) {
    const int f = i / ((TR - Bt) * kRS), r = i % ((TR - Bt) * kRS);
    Zs[f * TR * kRS + Bt * kRS + r] = 0.0;  // padding rows of the lift k-steps stay zero
  }
  if (threadIdx.x == 0) mbar_init(bar, 1);
  __syncthreads();
  unsigned phase = 0;
  constexpr unsigned kTBytes = 2 * Bt * kRS * sizeof(double);
  for (int64_t it = blockIdx.x; it < prm.ntiles; it += gridDim.x) {
    const int64_t tile = prm.tile0 + it;
    double* Qt = prm.Q + tile * B * kRS;
    const double* gtr = prm.traces + tile * 4 * Bt * kRS;
    if (threadIdx.x == 0 && it + gridDim.x < prm.ntiles) {
      const int64_t nt = tile + gridDim.x;
      prefetch_l2(prm.traces + nt * 4 * Bt * kRS, 4 * Bt * kRS * sizeof(double));
      prefetch_l2(prm.aplus + nt * 4 * kP * kP * kL, 4 * kP * kP * kL * sizeof(double));
      prefetch_l2(prm.aminus + nt * 4 * kP * kP * kL, 4 * kP * kP * kL * sizeof(double));
      prefetch_l2(prm.Q + nt * B * kRS, B * kRS * sizeof(double));
    }
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {
      // 1. all loads of the pass in flight at once
      if (threadIdx.x == 0) {
        mbar_expect_tx(bar, kTBytes);
        bulk_g2s(Ts, gtr + 2 * pass * Bt * kRS, kTBytes, bar);
      }
      int hh[2];
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        const int F = 2 * pass + f;
        const int64_t slot = (tile * 4 + F) * kL + x.lane;
        const int64_t nbe = prm.nb[slot];
        const int jh = prm.jh[slot];
        hh[f] = jh >> 2;
        const double* src = prm.traces + (((nbe >> 5) * 4 + (jh & 3)) * Bt) * kRS + x.p * kL + (nbe & 31);
        double* Z = Zs + f * TR * kRS;
#pragma unroll
        for (int n = 0; n < Bt; ++n) cp_async8(Z + swz(n, col), src + n * kRS);
      }
      double ap[2][kP], am[2][kP];
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        const int64_t fo = ((tile * 4 + 2 * pass + f) * kP + x.p) * kP * kL + x.lane;
#pragma unroll
        for (int q = 0; q < kP; ++q) {
          ap[f][q] = prm.aplus[fo + q * kL];
          am[f][q] = prm.aminus[fo + q * kL];
        }
      }
      cp_async_wait_all();
      // 2. rotate the own column of Z in place: z = f^h t
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        double* Z = Zs + f * TR * kRS;
        double tn[Bt];
#pragma unroll
        for (int n = 0; n < Bt; ++n) tn[n] = Z[swz(n, col)];
        Gen<N>::template rot<double>(hh[f], tn, [&](int m, double z) { Z[swz(m, col)] = z; });
      }
      mbar_wait(bar, phase);
      phase ^= 1;
      __syncthreads();
      // 3. Y = T A+^T + Z A-^T per element
      double y[2][Bt];
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        const double* Z = Zs + f * TR * kRS;
        const double* T = Ts + f * Bt * kRS + x.lane;
#pragma unroll
        for (int m = 0; m < Bt; ++m) {
          double sacc = 0.0;
#pragma unroll
          for (int q = 0; q < kP; ++q)
            sacc = fma(T[m * kRS + q * kL], ap[f][q], fma(Z[swz(m, q * kL + x.lane)], am[f][q], sacc));
          y[f][m] = sacc;
        }
      }
      __syncthreads();  // all columns of Z and T read
#pragma unroll
      for (int f = 0; f < 2; ++f)
#pragma unroll
        for (int m = 0; m < Bt; ++m) Zs[f * TR * kRS + swz(m, col)] = y[f][m];
      __syncwarp();
      // 4. lift with the DMMA tiles of R^i, update Q
      double acc[G::QMT][4][2];
      zero_acc(acc);
      if (pass == 0) {
        G::template lift<0>(x, Zs, acc);
        G::template lift<1>(x, Zs + TR * kRS, acc);
      } else {
        G::template lift<2>(x, Zs, acc);
        G::template lift<3>(x, Zs + TR * kRS, acc);
      }
#if YDG_QSTAGE
      __syncthreads();  // Y consumed by every warp: stage the update over Z and T
      stage_acc<G::QMT, B>(x, smem, acc);
      __syncthreads();
      update_q<B>(Qt, smem);
#else
      add_q<G::QMT, B>(x, Qt, acc);
#endif
      __syncthreads();  // before the next pass overwrites Z and T
    }
  }
}

}  // namespace dm
}  // namespace ydg
