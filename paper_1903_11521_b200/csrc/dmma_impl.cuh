// FP64 tensor-core (DMMA m8n8k4) kernels of the ADER-DG update (sm_100a, fp64, P = 9).
//
// Data of a 32-element tile live in shared memory as [row][col] with col = p*32 + e
// (quantity-major), rows swizzled (col ^ 8*(row & 1)) so that the 4-row x 8-column DMMA
// B-fragment loads take the minimum two wavefronts.  A tile is kL = 8 (or 16) elements; a
// CTA has 3 (6) warps and 4 (2) CTAs share an SM, so each SM sub-partition runs three warps
// (equal load on the four tensor pipes) and one CTA's barriers, memory phases and latency
// chains overlap the others' DMMAs.  Warp w owns the 8-column tiles (quantity 3g + k,
// elements 8ct..8ct+7), k = 0..2, with g = w / kCT, ct = w % kCT -- its "units".  Every B operand a warp feeds to a
// DMMA is warp-private; only the per-element quantity mixing (star matrices A*, flux
// solvers) reads other warps' columns.  Global matrices are the DMMA A operands:
// generated 8x4 tiles over freely grouped rows (gen/dmma.py, gen/tiling.py).
//
// Face traces T_i = R^iT I live in HBM as [tile][face][lane][TS] with an element-face
// block [m][q] of TS = even(9*Bt) doubles: the producer writes a face of a tile with one
// TMA bulk store, the consumer gathers a neighbour's face with one TMA bulk copy.
#pragma once
#include "kernels.cuh"
#include "setup.h"

namespace ydg {
namespace dm {

constexpr int kP = 9;
constexpr int kL = kDmLanes;   // elements per tile (HBM layouts of the fp64 path use the same)
constexpr int kRS = kP * kL;   // columns per row
constexpr int kCT = kL / 8;    // 8-element column tiles per quantity
constexpr int kJH = kL < 16 ? 16 : kL;  // bytes of j|h per (tile, face) (padded for TMA)
constexpr int kW = kDmWarps;   // warps per CTA (kDmCtasPerSm CTAs per SM: 3 warps per sub-partition)
constexpr int kT = kW * 32;    // threads per CTA
constexpr int kU = 3;          // units (8-column tiles) per warp
// warp-private X buffer: [c][k][row][8 elements], (c, k) blocks kXS doubles apart.  The
// star-chunk stores of lanes xk = 0, 1, 2 hit the same 16 banks at a block stride of 32
// doubles (3 wavefronts per store); YDG_XPAD = 8 puts block k + 1 on the other half (2)
#ifndef YDG_XPAD
#define YDG_XPAD 0
#endif
constexpr int kXS = 4 * 8 + YDG_XPAD;
constexpr int kXW = 3 * kU * kXS;
#ifndef YDG_XBUF
#define YDG_XBUF 1
#endif
constexpr int kXBUF = YDG_XBUF;      // star-chunk buffers per warp (1: reuse after __syncwarp)

enum Src { SRC_Q, SRC_S, SRC_I };

// Row swizzle inside aligned 8-column groups so that a 4-row x 8-column B-fragment load hits
// 4 disjoint bank groups: rows of 144 doubles (16-element tiles) start on the same bank ->
// XOR 8 on odd rows; rows of 72 doubles (8-element tiles) alternate by 8 banks already ->
// XOR 4 on rows 2, 3 (mod 4).  Column pairs (2c, 2c+1) stay adjacent.
__device__ __forceinline__ int swz(int row, int col) {
  return row * kRS + (kL == 16 ? (col ^ ((row & 1) << 3)) : (col ^ ((row & 2) << 1)));
}

struct Ctx {
  int lane, w;
  int col0;           // column of unit 0 of this warp's B fragments / C fragments: 3g*32 + 8ct
  int sh4, sh8;       // 8 * (lane & 3), 8 * (lane >> 2): byte of a k-set / m-tile row word
  int qcol0;          // flux kernel: HBM column of unit 0 of this warp's C fragments
  // star chunk role: lane -> (element xe = 8ct + (lane & 7), unit xk = lane >> 3; xk = 3 idle)
  int xe, xk;
  // column role (sparse DFMA steps): thread cc < 9 kL owns data column cc = cp*kL + ce
  int cc, ce, cp;
  // tail role (warp-synchronous CK tail): element te = 3 w + lane / 9, quantity tp = lane % 9,
  // column tc = tp*kL + te, or -1 if the lane has no element
  int te, tp, tc;
  const double* star;  // star matrices of this tile, global [c][p][3][kL]
  double* S;          // [SROWS][288]  D^d, d >= 1
  double* I;          // [IROWS][288]  time integral rows < IROWS
  double* xb;         // warp-private [3][kU][4][8]
  double* xb2;        // second star-chunk buffer of CK step 0 (YDG_GEN_XPIPE): S rows >= B - IROWS
  const double* Qt;   // Q of this tile in global memory: [B][9][32]
  const double* frags;
  const double* fs;   // shared-memory A-fragment buffer (products staged there)
  unsigned long long* fbar;  // its mbarrier
  double a[9];        // star matrices, row p = 3g + xk: a[3c + j] = A*^c[p][q_j]
  int q0, q1, q2;     // star columns of row p
  double dt;
  int tid, grp;       // thread index within the (group of the) CTA, group index
  int shcap;          // grouped local kernel: fragments held in the shared buffer
  bool lfs;           // flux: the lift's A fragments are staged in shared memory (x.fs)
  __device__ __forceinline__ void sync() const {  // barrier of the thread's group
    if (kLocalGroups == 1) __syncthreads();
    else asm volatile("bar.sync %0, %1;" ::"r"(grp + 1), "n"(kT) : "memory");
  }
  const double* scal;  // kernel-parameter space: dt/(d+1) at [d], dt/(d+2) at [N + d]
  int N;
};

// Phase timing of the local kernel (build with YDG_NVFLAGS=-DYDG_PHASES): CTA 0, thread 0
// prints clock64 deltas of a few tiles.
#ifdef YDG_PHASES
#define YDG_PHASE(k) \
  do {               \
    if (threadIdx.x == 0 && blockIdx.x == 0) ph_t[k] = clock64(); \
  } while (0)
__device__ long long ph_t[16];
#else
#define YDG_PHASE(k) \
  do {               \
  } while (0)
#endif

template <int N>
struct DG;
template <int N>
__device__ const double* frag_table();
template <int N>
__device__ const double* fh_table();

// A fragments: read-only, reused by every warp and tile -> keep in L1 (evict_last); other
// streaming loads use evict_first so they do not push the fragment table out.
__device__ __forceinline__ double afrag_g(const Ctx& x, int tid) {
  double v;
  asm("ld.global.nc.L1::evict_last.f64 %0, [%1];" : "=d"(v) : "l"(x.frags + tid * 32 + x.lane));
  return v;
}
__device__ __forceinline__ double afrag_s(const Ctx& x, int i) { return x.fs[i * 32 + x.lane]; }
// table slot tid: the grouped local kernel holds slots [0, shcap) in shared memory
__device__ __forceinline__ double afrag(const Ctx& x, int tid) {
  if constexpr (kLocalGroups > 1) return tid < x.shcap ? afrag_s(x, tid) : afrag_g(x, tid);
  return afrag_g(x, tid);
}
// Products whose fragments may be staged in shared memory: CK step 0 and the volume term
// (local kernel), the lift (flux kernel).  With two CTAs per SM there is no room: off.
#ifndef YDG_LOCAL_FS
#define YDG_LOCAL_FS 0
#endif
#ifndef YDG_FLUX_FS
#define YDG_FLUX_FS 0
#endif
constexpr bool kLocalFs = YDG_LOCAL_FS && kLocalGroups == 1, kFluxFs = YDG_FLUX_FS || kFluxGroups > 1;
// capacity of the local kernel's fragment buffer (fragments of 256 B; the rest of the
// product reads the global table)
#ifndef YDG_LOCAL_FS_CAP
#define YDG_LOCAL_FS_CAP 56
#endif
constexpr int kLocalFsCap = YDG_LOCAL_FS_CAP;
// g: table index; r: index within the product's staged region.  The grouped kernel holds
// table slots [0, shcap) (CK step 0, then the volume) in a static shared buffer.
__device__ __forceinline__ double afrag_l(const Ctx& x, int g, int r) {
  if constexpr (kLocalGroups > 1) return afrag(x, g);
  return (kLocalFs && r < kLocalFsCap) ? afrag_s(x, r) : afrag_g(x, g);
}
__device__ __forceinline__ double afrag_f(const Ctx& x, int g, int r) {
  return (kFluxFs && x.lfs) ? afrag_s(x, r) : afrag_g(x, g);
}
// L2 eviction hints on the streaming stores (bit mask, build flag): 1 = trace bulk stores of
// the local kernel, 2 = its Q stores, 4 = the flux kernel's Q stores -- evict_first, so that
// the Q^n rows a tile re-reads stay in L2
#ifndef YDG_L2HINT
#define YDG_L2HINT 3  // measured: local 15.31 -> 14.77-14.95 ms (c1); 7 (also flux Q stores) slows the flux kernel
#endif
__device__ __forceinline__ unsigned long long evict_first_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
template <int BIT>
__device__ __forceinline__ void st_q2(double* p, double2 v) {
  if constexpr ((YDG_L2HINT & BIT) != 0) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y),
                 "l"(evict_first_policy())
                 : "memory");
  } else {
    *reinterpret_cast<double2*>(p) = v;
  }
}
// Coherent (not .nc): in the fused kernel the tile's Q was written by its own flux phase
// earlier in the same launch, which the non-coherent read-only path need not observe.
__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm volatile("ld.global.L1::evict_first.f64 %0, [%1];" : "=d"(v) : "l"(p));  // volatile: kept after the barriers
  return v;
}
// star matrices of the tile: read by the star-chunk role at the tile start and again by every
// sparse-DFMA CK step; YDG_STAR_L1=1 keeps them in L1 (evict_last) between the reads
#ifndef YDG_STAR_L1
#define YDG_STAR_L1 0
#endif
__device__ __forceinline__ double ld_star(const double* p) {
  if constexpr (YDG_STAR_L1 == 0) return ld_stream(p);
  double v;
  asm("ld.global.nc.L1::evict_last.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ int krow(const Ctx& x, unsigned w) { return static_cast<int>((w >> x.sh4) & 0xffu); }
__device__ __forceinline__ int mrow(const Ctx& x, unsigned long long w) {
  return static_cast<int>((w >> x.sh8) & 0xffull);
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}
__device__ __forceinline__ void dmma3(double (&acc)[kU][2], double a, const double (&bf)[kU]) {
#pragma unroll
  for (int k = 0; k < kU; ++k) dmma(acc[k], a, bf[k]);
}

template <int MT>
__device__ __forceinline__ void zero_acc(double (&acc)[MT][kU][2]) {
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int c = 0; c < kU; ++c) acc[m][c][0] = acc[m][c][1] = 0.0;
}
// column of the B-fragment entry of unit k held by this lane (element 8ct + lane / 4)
__device__ __forceinline__ int bcol(const Ctx& x, int k) { return x.col0 + k * kL + (x.lane >> 2); }
// first of the two C-fragment columns of unit k held by this lane (elements 8ct + 2(lane & 3) + {0,1})
__device__ __forceinline__ int ccol(const Ctx& x, int k) { return x.col0 + k * kL + 2 * (x.lane & 3); }

template <Src SRC, int B>
__device__ __forceinline__ double load_data(const Ctx& x, int row, int col) {
  // Q^n of the tile is staged in shared memory at the rows of I (rows >= IROWS continue
  // into S) for the first CK step
  if constexpr (SRC == SRC_Q) return x.I[swz(row, col)];
  else if constexpr (SRC == SRC_S) return x.S[swz(row, col)];
  else return x.I[swz(row, col)];
}

// X^c = D A*^cT for the 4 rows r0..r3 (compile-time, uniform over the warp): lane
// (xe, xk) computes its element's column of quantity 3g + xk into the warp-private buffer
// buf ([c][k][r][8]); after a __syncwarp() xb_b reads one c's B fragments for the warp's
// three units.
template <Src SRC, int B>
__device__ __forceinline__ void xcalc(Ctx& x, int buf, int r0, int r1, int r2, int r3) {
  if (kXBUF == 1) __syncwarp();  // every lane has read the previous chunk's B fragments
  if (x.xk < kU) {
    double* xb = x.xb + (buf % kXBUF) * kXW;
    const int rr[4] = {r0, r1, r2, r3};
    // all 12 loads first (no store in between), then 12 independent 3-term dot products:
    // three dependent FP64 waves instead of a chain per row (the FP64 pipe is shared with
    // the queued DMMAs, so every dependent FP64 step waits behind them)
    double d[4][3];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      d[r][0] = load_data<SRC, B>(x, rr[r], x.q0 * kL + x.xe);
      d[r][1] = load_data<SRC, B>(x, rr[r], x.q1 * kL + x.xe);
      d[r][2] = load_data<SRC, B>(x, rr[r], x.q2 * kL + x.xe);
    }
    double v[4][3];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) v[r][c] = x.a[3 * c] * d[r][0];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) v[r][c] = fma(x.a[3 * c + 1], d[r][1], v[r][c]);
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) v[r][c] = fma(x.a[3 * c + 2], d[r][2], v[r][c]);
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) xb[(c * kU + x.xk) * kXS + r * 8 + (x.lane & 7)] = v[r][c];
  }
}
// Pipelined form (generator YDG_GEN_XPIPE, CK step 0): the chunk of k-set i + 1 is computed
// in the same basic block as k-set i's DMMAs, into the other of two buffers (x.xb, x.xb2),
// so that its dependent FP64 waves interleave with those DMMAs.  No branch: lanes xk = 3
// compute unit 2's values again and only their stores are predicated off.
template <Src SRC, int B>
__device__ __forceinline__ void xcalc_to(const Ctx& x, double* xb, int r0, int r1, int r2, int r3) {
  const int rr[4] = {r0, r1, r2, r3};
  double d[4][3];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    d[r][0] = load_data<SRC, B>(x, rr[r], x.q0 * kL + x.xe);
    d[r][1] = load_data<SRC, B>(x, rr[r], x.q1 * kL + x.xe);
    d[r][2] = load_data<SRC, B>(x, rr[r], x.q2 * kL + x.xe);
  }
  double v[4][3];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) v[r][c] = x.a[3 * c] * d[r][0];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) v[r][c] = fma(x.a[3 * c + 1], d[r][1], v[r][c]);
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) v[r][c] = fma(x.a[3 * c + 2], d[r][2], v[r][c]);
  const bool st = x.xk < kU;
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      if (st) xb[(c * kU + x.xk) * kXS + r * 8 + (x.lane & 7)] = v[r][c];
}
__device__ __forceinline__ void xb_from(const double* xb, const Ctx& x, int c, double (&bf)[kU]) {
#pragma unroll
  for (int k = 0; k < kU; ++k) bf[k] = xb[(c * kU + k) * kXS + (x.lane & 3) * 8 + (x.lane >> 2)];
}
__device__ __forceinline__ void xb_b(const Ctx& x, int buf, int c, double (&bf)[kU]) {
  const double* xb = x.xb + (buf % kXBUF) * kXW;
#pragma unroll
  for (int k = 0; k < kU; ++k) bf[k] = xb[(c * kU + k) * kXS + (x.lane & 3) * 8 + (x.lane >> 2)];
}

// Gathered B fragments of the own quantity column: lane row = byte (lane & 3) of w.
__device__ __forceinline__ void ismem_b(const Ctx& x, unsigned w, double (&bf)[kU]) {
  const int row = krow(x, w);
#pragma unroll
  for (int k = 0; k < kU; ++k) bf[k] = x.I[swz(row, bcol(x, k))];
}
// rows >= IROWS of the time integral are dt * Q (only D^0 contributes), from global memory
template <int B>
__device__ __forceinline__ void gq_b(const Ctx& x, unsigned w, double (&bf)[kU]) {
  const int row = krow(x, w);
#pragma unroll
  for (int k = 0; k < kU; ++k) bf[k] = x.dt * ld_stream(x.Qt + row * kRS + bcol(x, k));
}
__device__ __forceinline__ void smem_b(const Ctx& x, const double* Y, unsigned w, double (&bf)[kU]) {
  const int row = krow(x, w);
#pragma unroll
  for (int k = 0; k < kU; ++k) bf[k] = Y[swz(row, bcol(x, k))];
}

// Write D^{d+1} = dt/(d+1) acc of one m-tile (rows from the word w) into S and accumulate
// the time integral; at d = 0 the integral starts from dt * Q.
template <int FIRST, int B>
__device__ __forceinline__ void ck_wb(Ctx& x, const double (&acc)[kU][2], int d, unsigned long long w) {
  const int row = mrow(x, w);
  if (row == 0xff) return;
  const double sc = x.scal[d], ic = x.scal[x.N + d];
#pragma unroll
  for (int k = 0; k < kU; ++k) {
    const int s = swz(row, ccol(x, k));
    const double v0 = sc * acc[k][0], v1 = sc * acc[k][1];
    *reinterpret_cast<double2*>(x.S + s) = make_double2(v0, v1);
    double2 i2 = *reinterpret_cast<const double2*>(x.I + s);
    if (FIRST) {
      i2 = make_double2(fma(ic, v0, x.dt * i2.x), fma(ic, v1, x.dt * i2.y));
    } else {
      i2.x = fma(ic, v0, i2.x);
      i2.y = fma(ic, v1, i2.y);
    }
    *reinterpret_cast<double2*>(x.I + s) = i2;
  }
}
// Rows [LO, HI) of the time-integral region receive no derivative: I = dt * Q.
template <int LO, int HI>
__device__ __forceinline__ void scale_irows(Ctx& x) {
  for (int i = x.tid; i < (HI - LO) * kRS; i += kT) {
    double* v = x.I + (LO + i / kRS) * kRS + i % kRS;
    *v = x.dt * *v;
  }
}

// Q += acc over all m-tiles (rows from the words w[]), two m-tiles per batch: the batch's
// Q loads are all issued before its stores (one L2/HBM latency per batch, bounded register
// use), values are added into the accumulators, then stored (16-byte, two elements).
// Qs: rows < IR of Q^n already in shared memory (plain [row][288] layout), else nullptr
template <int MT, int IR>
__device__ __forceinline__ void q_batch(const Ctx& x, const double* Qt, const double* Qs,
                                        const unsigned long long (&w)[MT], int m0, double2 (&v)[2][kU]) {
#pragma unroll
  for (int k2 = 0; k2 < 2; ++k2) {
    const int row = m0 + k2 < MT ? mrow(x, w[m0 + k2 < MT ? m0 + k2 : 0]) : 0xff;
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      if (row == 0xff) v[k2][k] = make_double2(0.0, 0.0);
      else if (row < IR) v[k2][k] = *reinterpret_cast<const double2*>(Qs + row * kRS + ccol(x, k));
      else v[k2][k] = *reinterpret_cast<const double2*>(Qt + row * kRS + ccol(x, k));
    }
  }
}
// Q += acc over all m-tiles (rows from the words w[]; rows < IR of Q^n are read from the
// shared copy Qs), two m-tiles per batch, software-pipelined: the next batch's Q loads are
// issued before the current batch's stores (one memory latency in total, bounded registers).
// global rows (>= IR) of the first batch, ahead of time (add_q's `pre`)
template <int MT, int IR>
__device__ __forceinline__ void q_pre(const Ctx& x, const double* Qt, const unsigned long long (&w)[MT],
                                      double2 (&v)[2][kU]) {
#pragma unroll
  for (int k2 = 0; k2 < 2; ++k2) {
    const int row = k2 < MT ? mrow(x, w[k2 < MT ? k2 : 0]) : 0xff;
#pragma unroll
    for (int k = 0; k < kU; ++k)
      v[k2][k] = (row == 0xff || row < IR) ? make_double2(0.0, 0.0)
                                           : *reinterpret_cast<const double2*>(Qt + row * kRS + ccol(x, k));
  }
}
template <int MT, int IR = 0>
__device__ __forceinline__ void add_q(const Ctx& x, double* Qt, double (&acc)[MT][kU][2],
                                      const unsigned long long (&w)[MT], const double* Qs = nullptr,
                                      const double2 (*pre)[kU] = nullptr) {
  double2 vc[2][kU], vn[2][kU];
  if (pre) {  // global rows preloaded; rows < IR from the shared copy
#pragma unroll
    for (int k2 = 0; k2 < 2; ++k2) {
      const int row = k2 < MT ? mrow(x, w[k2 < MT ? k2 : 0]) : 0xff;
#pragma unroll
      for (int k = 0; k < kU; ++k)
        vc[k2][k] = (row != 0xff && row < IR) ? *reinterpret_cast<const double2*>(Qs + row * kRS + ccol(x, k))
                                              : pre[k2][k];
    }
  } else {
    q_batch<MT, IR>(x, Qt, Qs, w, 0, vc);
  }
#pragma unroll
  for (int m0 = 0; m0 < MT; m0 += 2) {
    if (m0 + 2 < MT) q_batch<MT, IR>(x, Qt, Qs, w, m0 + 2, vn);
#pragma unroll
    for (int k2 = 0; k2 < 2; ++k2) {
      if (m0 + k2 >= MT) continue;
      const int row = mrow(x, w[m0 + k2]);
      if (row == 0xff) continue;
#pragma unroll
      for (int k = 0; k < kU; ++k)
        st_q2<2>(Qt + row * kRS + ccol(x, k),
                 make_double2(acc[m0 + k2][k][0] + vc[k2][k].x, acc[m0 + k2][k][1] + vc[k2][k].y));
    }
    if (m0 + 2 < MT) {
#pragma unroll
      for (int k2 = 0; k2 < 2; ++k2)
#pragma unroll
        for (int k = 0; k < kU; ++k) vc[k2][k] = vn[k2][k];
    }
  }
}

// Q rows of two m-tiles (words w0, w1; ~0 = absent) for the m-tile-group lift: load_q2
// issues the loads, store_q2 writes Q + acc.
__device__ __forceinline__ void load_q2(const Ctx& x, const double* Qt, unsigned long long w0, unsigned long long w1,
                                        double2 (&q)[2][kU]) {
#pragma unroll
  for (int k2 = 0; k2 < 2; ++k2) {
    const int row = mrow(x, k2 ? w1 : w0);
#pragma unroll
    for (int k = 0; k < kU; ++k)
      q[k2][k] = row == 0xff ? make_double2(0.0, 0.0) : *reinterpret_cast<const double2*>(Qt + row * kRS + ccol(x, k));
  }
}
__device__ __forceinline__ void copy_q2(const double2 (&a)[2][kU], double2 (&b)[2][kU]) {
#pragma unroll
  for (int k2 = 0; k2 < 2; ++k2)
#pragma unroll
    for (int k = 0; k < kU; ++k) b[k2][k] = a[k2][k];
}
__device__ __forceinline__ void store_q2(const Ctx& x, double* Qt, unsigned long long w0, unsigned long long w1,
                                         const double (&acc)[2][kU][2], const double2 (&q)[2][kU]) {
#pragma unroll
  for (int k2 = 0; k2 < 2; ++k2) {
    const int row = mrow(x, k2 ? w1 : w0);
    if (row == 0xff) continue;
#pragma unroll
    for (int k = 0; k < kU; ++k)
      *reinterpret_cast<double2*>(Qt + row * kRS + ccol(x, k)) =
          make_double2(q[k2][k].x + acc[k2][k][0], q[k2][k].y + acc[k2][k][1]);
  }
}

// ---- flux-kernel layout: CTAs of kLF = 8 elements (half of a 16-element HBM tile), 3 warps,
// four CTAs per SM.  Shared rows have 72 columns; warp w owns units (quantity 3w + k, the
// CTA's 8 elements); Q columns in HBM are (3w + k) * kL + half * 8 + element.
constexpr int kLF = 8;
constexpr int kRSF = kP * kLF;
constexpr int kWF = 3;
constexpr int kTF = kWF * 32;
constexpr int kHalves = kL / kLF;
constexpr int kFluxCtas = 4;
#ifndef YDG_FLUX_LATE_OWN
#define YDG_FLUX_LATE_OWN 0
#endif
constexpr bool kFluxLateOwn = YDG_FLUX_LATE_OWN;
// YDG_FLUX_PF: L2 prefetch of the next unit's neighbour (bit 1) / own (bit 2) face blocks,
// issued at face YDG_FLUX_PF_FACE of the current unit
#ifndef YDG_FLUX_PF
#define YDG_FLUX_PF 0
#endif
#ifndef YDG_FLUX_PF_FACE
#define YDG_FLUX_PF_FACE 1
#endif
constexpr int kFluxPf = YDG_FLUX_PF, kFluxPfFace = YDG_FLUX_PF_FACE;
// face of the current unit at which the next unit's Q is prefetched into L2 (-1: none)
#ifndef YDG_FLUX_QPF_FACE
#define YDG_FLUX_QPF_FACE 3
#endif
constexpr int kFluxQpfFace = YDG_FLUX_QPF_FACE;
#ifndef YDG_VOL_QEARLY
#define YDG_VOL_QEARLY 0  // measured (c1 local): 1 spills (468 B) and runs 14.47 vs 13.74 ms
#endif
#ifndef YDG_FLUX_QEARLY
#define YDG_FLUX_QEARLY 2  // measured (c1 flux): 0: 7.54, 1: 7.27, 2: 7.19-7.22 ms
#endif
constexpr int kFluxQEarly = YDG_FLUX_QEARLY;
__device__ __forceinline__ int swzf(int row, int col) { return row * kRSF + (col ^ ((row & 2) << 1)); }
__device__ __forceinline__ void smem_bf(const Ctx& x, const double* Y, unsigned w, double (&bf)[kU]) {
  const int row = krow(x, w);
#pragma unroll
  for (int k = 0; k < kU; ++k) bf[k] = Y[swzf(row, x.col0 + k * kLF + (x.lane >> 2))];
}
__device__ __forceinline__ int qcolf(const Ctx& x, int k) { return x.qcol0 + k * kL + 2 * (x.lane & 3); }
// Q rows of the flux kernel's read-modify-write (coherent loads: the first pair's update
// is re-read by the second); YDG_FLUX_QNA=1: L1 no-allocate
__device__ __forceinline__ double2 ld_q2(const double* p) {
#if defined(YDG_FLUX_QNA) && YDG_FLUX_QNA
  double2 v;
  asm volatile("ld.global.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
#else
  return *reinterpret_cast<const double2*>(p);
#endif
}
__device__ __forceinline__ void load_qf(const Ctx& x, const double* Qt, unsigned long long w0, unsigned long long w1,
                                        double2 (&q)[2][kU]) {
#pragma unroll
  for (int k2 = 0; k2 < 2; ++k2) {
    const int row = mrow(x, k2 ? w1 : w0);
#pragma unroll
    for (int k = 0; k < kU; ++k)
      q[k2][k] = row == 0xff ? make_double2(0.0, 0.0) : ld_q2(Qt + row * kRS + qcolf(x, k));
  }
}
__device__ __forceinline__ void store_qf(const Ctx& x, double* Qt, unsigned long long w0, unsigned long long w1,
                                         const double (&acc)[2][kU][2], const double2 (&q)[2][kU]) {
#pragma unroll
  for (int k2 = 0; k2 < 2; ++k2) {
    const int row = mrow(x, k2 ? w1 : w0);
    if (row == 0xff) continue;
#pragma unroll
    for (int k = 0; k < kU; ++k)
      st_q2<4>(Qt + row * kRS + qcolf(x, k), make_double2(q[k2][k].x + acc[k2][k][0], q[k2][k].y + acc[k2][k][1]));
  }
}

// Trace C fragments of one m-tile -> staging block [lane][m][q] (stride TS per lane).
template <int TS>
__device__ __forceinline__ void stage_trace(const Ctx& x, double* stg, const double (&acc)[kU][2], unsigned long long w) {
  const int m = mrow(x, w);
  if (m == 0xff) return;
  const int e = (x.col0 % kL) + 2 * (x.lane & 3), p0 = x.col0 / kL;
#pragma unroll
  for (int k = 0; k < kU; ++k) {
    stg[e * TS + m * kP + p0 + k] = acc[k][0];
    stg[(e + 1) * TS + m * kP + p0 + k] = acc[k][1];
  }
}

// Flux of the Godunov state of one face-basis row (P:1341-1342 with reading R8):
//   y = A+ t + A- z  for the own state t and the rotated neighbour state z (quantity order
//   sxx syy szz sxy syz sxz u v w), rebuilt from the factored solver c (setup.h):
//   tractions tau = sigma n; normal (p-wave) and tangential (s-wave) interface states
//   v*_n = v_n- + Z+/S dv_n + dtau_n/S,  tau*_n = tau_n- + Z-/S dtau_n + Z-Z+/S dv_n (per wave
//   type, S = Z- + Z+); flux  sigma = -lam v*_n I - mu (n v*^T + v* n^T),  v = -tau*/rho, all
//   times -2|S_i|/det J.  Same linear map as T A_x(m-) G-+ T^-1 (setup.cpp), ~80 FMAs
//   instead of 162.
__device__ __forceinline__ void godunov_flux(const double* t, const double* z, const double (&c)[kFaceCoeffs],
                                             double (&y)[kP]) {
  const double nx = c[0], ny = c[1], nz = c[2];
  const double t1x = fma(t[5], nz, fma(t[3], ny, t[0] * nx));
  const double t1y = fma(t[4], nz, fma(t[1], ny, t[3] * nx));
  const double t1z = fma(t[2], nz, fma(t[4], ny, t[5] * nx));
  const double t2x = fma(z[5], nz, fma(z[3], ny, z[0] * nx));
  const double t2y = fma(z[4], nz, fma(z[1], ny, z[3] * nx));
  const double t2z = fma(z[2], nz, fma(z[4], ny, z[5] * nx));
  const double dvx = z[6] - t[6], dvy = z[7] - t[7], dvz = z[8] - t[8];
  const double dtx = t2x - t1x, dty = t2y - t1y, dtz = t2z - t1z;
  const double vn1 = fma(t[8], nz, fma(t[7], ny, t[6] * nx));
  const double dvn = fma(dvz, nz, fma(dvy, ny, dvx * nx));
  const double tn1 = fma(t1z, nz, fma(t1y, ny, t1x * nx));
  const double dtn = fma(dtz, nz, fma(dty, ny, dtx * nx));
  // p wave: normal components
  const double vns = fma(c[5], dtn, fma(1.0 - c[3], dvn, vn1));
  const double tns = fma(c[4], dvn, fma(c[3], dtn, tn1));
  // s wave: whole vectors, normal parts replaced below
  const double bs = 1.0 - c[6];
  const double vsx = fma(c[8], dtx, fma(bs, dvx, t[6]));
  const double vsy = fma(c[8], dty, fma(bs, dvy, t[7]));
  const double vsz = fma(c[8], dtz, fma(bs, dvz, t[8]));
  const double tsx = fma(c[7], dvx, fma(c[6], dtx, t1x));
  const double tsy = fma(c[7], dvy, fma(c[6], dty, t1y));
  const double tsz = fma(c[7], dvz, fma(c[6], dtz, t1z));
  const double cv = vns - fma(vsz, nz, fma(vsy, ny, vsx * nx));
  const double ct = tns - fma(tsz, nz, fma(tsy, ny, tsx * nx));
  const double vx = fma(cv, nx, vsx), vy = fma(cv, ny, vsy), vz = fma(cv, nz, vsz);
  const double tx = fma(ct, nx, tsx), ty = fma(ct, ny, tsy), tz = fma(ct, nz, tsz);
  const double L = c[9] * vns, M = c[10], M2 = 2.0 * c[10], R = c[11];
  y[0] = -fma(M2 * nx, vx, L);
  y[1] = -fma(M2 * ny, vy, L);
  y[2] = -fma(M2 * nz, vz, L);
  y[3] = -M * fma(nx, vy, ny * vx);
  y[4] = -M * fma(ny, vz, nz * vy);
  y[5] = -M * fma(nx, vz, nz * vx);
  y[6] = -R * tx;
  y[7] = -R * ty;
  y[8] = -R * tz;
}

// Column role (sparse DFMA CK steps): star coefficients of quantity cp of element ce.
__device__ __forceinline__ void col_star(const Ctx& x, int ce, int cp, double (&ca)[9], int& q0, int& q1, int& q2) {
  constexpr unsigned long long packed[9] = {6 | 7 << 5 | 8 << 10, 6 | 7 << 5 | 8 << 10, 6 | 7 << 5 | 8 << 10,
                                            6 | 7 << 5 | 7 << 10, 7 | 8 << 5 | 8 << 10, 6 | 8 << 5 | 8 << 10,
                                            0 | 3 << 5 | 5 << 10, 3 | 1 << 5 | 4 << 10, 5 | 4 << 5 | 2 << 10};
  unsigned long long w = 0;
#pragma unroll
  for (int i = 0; i < 9; ++i) w = (cp == i) ? packed[i] : w;
  q0 = static_cast<int>(w & 31);
  q1 = static_cast<int>((w >> 5) & 31);
  q2 = static_cast<int>((w >> 10) & 31);
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int j = 0; j < 3; ++j) ca[3 * c + j] = ld_star(x.star + ((c * kP + cp) * 3 + j) * kL + ce);
}
template <Src SRC, int B>
__device__ __forceinline__ void col_x(const Ctx& x, int l, int ce, const double (&ca)[9], int q0, int q1, int q2,
                                      double& x0, double& x1, double& x2) {
  const double d0 = load_data<SRC, B>(x, l, q0 * kL + ce);
  const double d1 = load_data<SRC, B>(x, l, q1 * kL + ce);
  const double d2 = load_data<SRC, B>(x, l, q2 * kL + ce);
  x0 = fma(ca[2], d2, fma(ca[1], d1, ca[0] * d0));
  x1 = fma(ca[5], d2, fma(ca[4], d1, ca[3] * d0));
  x2 = fma(ca[8], d2, fma(ca[7], d1, ca[6] * d0));
}
// Write-back of a sparse CK step: D^{d+1} = dt/(d+1) y into S, time integral (as ck_wb).
template <int FIRST, int BO>
__device__ __forceinline__ void col_wb(Ctx& x, int cc, const double (&y)[BO], int d) {
  const double sc = x.scal[d], ic = x.scal[x.N + d];
#pragma unroll
  for (int k = 0; k < BO; ++k) {
    const int s = swz(k, cc);
    const double v = sc * y[k];
    x.S[s] = v;
    x.I[s] = FIRST ? fma(ic, v, x.dt * x.I[s]) : fma(ic, v, x.I[s]);
  }
}

template <int N>
struct Layout {
  using G = DG<N>;
  static constexpr int XB = kXBUF * kW * kXW;  // doubles (star-chunk buffers)
  static constexpr int FACE = kL * G::TS;      // doubles of one face of a tile
  // local kernel: [I][S][xb]; Q^n of the tile is staged over I and S for the first CK
  // step; the two trace staging blocks reuse S and xb
  static constexpr int ROWS = (G::IROWS + G::SROWS > G::B ? G::IROWS + G::SROWS : G::B);
  // A-fragment buffer (CK step 0, then the volume term) after I, S, xb and the staging
  static constexpr int FOFF = (ROWS * kRS + XB > G::IROWS * kRS + 2 * FACE ? ROWS * kRS + XB
                                                                           : G::IROWS * kRS + 2 * FACE);
  static constexpr int FSMAX0 = G::CK0_NF > G::VOL_NF ? G::CK0_NF : G::VOL_NF;
  static constexpr int FSMAX = kLocalFs ? (FSMAX0 < kLocalFsCap ? FSMAX0 : kLocalFsCap) : 0;
  static constexpr int LOCAL = FOFF + FSMAX * 32 + 2;  // + two mbarriers
  static constexpr int LOCALG = (LOCAL + 15) & ~15;     // one group's region (grouped kernel)
  // grouped kernel: CK step 0's fragments, then the volume's, as many as fit in 227 KB
  static constexpr int LSH0 = (227 * 1024 / 8 - kLocalGroups * LOCALG) / 32;
  // (shared slots = the first table slots: CK step 0's fragments, the volume's next, then
  // the traces'; the flux kernel's lift fragments follow all of them)
  static constexpr int LSH = kLocalGroups == 1 ? 0 : (LSH0 < G::LIFT_F0 ? LSH0 : G::LIFT_F0);
  static constexpr int LOCALCTA = kLocalGroups == 1 ? LOCAL : kLocalGroups * LOCALG + LSH * 32;
  // flux kernel (8-element CTAs): own face block, neighbour blocks, two Y buffers,
  // coefficients, slots, j|h, mbarriers
  static constexpr int FACEF = kLF * G::TS;  // doubles of one face of a flux CTA
  static constexpr int FLUX = 2 * FACEF + 2 * G::Bt * kRSF + kFaceCoeffs * kLF + 16 + 2;  // + slots, j|h, mbarriers
  static constexpr int FLUXG = (FLUX + 15) & ~15;  // one group's region (128-byte aligned)
  static constexpr int FLUXCTA = kFluxGroups * FLUXG + (kFluxFs ? G::LIFT_NF * 32 : 0);
  // fused kernel (dm_fused: flux of the previous step, then the local part, per tile): a
  // group region holds either phase's buffers (FOFF doubles of the local part, FLUXDATA of
  // the flux part), then four mbarriers (local: fragments, Q rows; flux: own, neighbour);
  // the shared A-fragment slots (CK step 0, the volume) take the rest of the 227 KB
  static constexpr int FLUXDATA = 2 * FACEF + 2 * G::Bt * kRSF + kFaceCoeffs * kLF + 16;
  static constexpr int FBAR = FOFF > FLUXDATA ? FOFF : FLUXDATA;
  static constexpr int FUSEDG = (FBAR + 4 + 15) & ~15;
  static constexpr int LSHF0 = (227 * 1024 / 8 - kLocalGroups * FUSEDG) / 32;
  static constexpr int LSHF = LSHF0 < G::LIFT_F0 ? LSHF0 : G::LIFT_F0;
  static constexpr int FUSEDCTA = kLocalGroups * FUSEDG + LSHF * 32;
};

// ---- asynchronous copy helpers (TMA bulk copies + mbarrier, Ampere-style cp.async)
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
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  if constexpr ((YDG_L2HINT & 1) != 0) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
                 "r"(smem_addr(src)), "r"(bytes), "l"(evict_first_policy())
                 : "memory");
  } else {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
                 "r"(bytes)
                 : "memory");
  }
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int K>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(K) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ void init_ctx(Ctx& x) {
  x.tid = threadIdx.x % kT;
  x.grp = threadIdx.x / kT;
  x.lane = x.tid & 31;
  x.w = x.tid >> 5;
  x.col0 = 3 * (x.w / kCT) * kL + 8 * (x.w % kCT);
  x.sh4 = 8 * (x.lane & 3);
  x.sh8 = 8 * (x.lane >> 2);
  x.xe = 8 * (x.w % kCT) + (x.lane & 7);
  x.xk = x.lane >> 3;
  x.cc = x.tid;
  x.ce = x.cc % kL;
  x.cp = x.cc / kL;
  x.te = 3 * x.w + x.lane / kP;
  x.tp = x.lane % kP;
  x.tc = (x.lane < 3 * kP && x.te < kL) ? x.tp * kL + x.te : -1;
}

// Stage NF A fragments starting at table index F0 into the shared buffer (one thread).
template <int N>
__device__ __forceinline__ void stage_frags(const Ctx& x, int F0, int NF) {
  mbar_expect_tx(x.fbar, NF * 32 * sizeof(double));
  bulk_g2s(const_cast<double*>(x.fs), frag_table<N>() + F0 * 32, NF * 32 * sizeof(double), x.fbar);
}
// Called by DG<N>::ck after CK step 0 (which ends with a barrier): the fragment buffer
// now receives the volume term's fragments.
// YDG_QPF bit 1: after CK step 0, the tile's Q^n rows >= IROWS (re-read by the traces and the
// volume's Q update, evicted from L2 since the staging) are prefetched into L2 again;
// bit 2: again before the volume term
#ifndef YDG_QPF
#define YDG_QPF 6  // measured (c1, 8-element tiles): 7: local 14.69 -> 14.11-14.19 ms, bit 1 alone 14.41;
                   // with the sparser derivative directions (shorter CK step 0): 7: 12.02-12.03,
                   // 6: 11.87-11.90, 4: 11.97-11.99, 5: 12.02-12.03, 3: 12.15-12.16, 2: 12.07-12.08 ms
#endif
template <int N>
__device__ __forceinline__ void after_ck0(Ctx& x) {
  if constexpr (kLocalFs)
    if (x.tid == 0) stage_frags<N>(x, DG<N>::VOL_F0, DG<N>::VOL_NF < kLocalFsCap ? DG<N>::VOL_NF : kLocalFsCap);
  if constexpr ((YDG_QPF & 1) != 0)
    if (x.tid == 32) prefetch_l2(x.Qt + DG<N>::IROWS * kRS, (DG<N>::B - DG<N>::IROWS) * kRS * sizeof(double));
}

// CK + time integral, face traces R^iT I (stored for the flux kernel) and
// the volume term for 32-element tiles.
template <int N>
__device__ __forceinline__ void flux_tile(Ctx& x, const StepParams<double>& prm, int64_t tile, double* smem,
                                          unsigned long long* bar, unsigned& ph_o, unsigned& ph_n);

// Body of the local kernel (FUSED = false) and of the fused step kernel (FUSED = true: each
// tile first receives the flux of the previous step from prm.traces_in -- flux_tile, the
// flux kernel's per-unit work -- then runs the local part, whose traces go to prm.traces).
template <int N, bool FUSED>
__device__ __forceinline__ void local_body(const StepParams<double>& prm) {
  using G = DG<N>;
  using Lay = Layout<N>;
  constexpr int B = G::B;
  constexpr int GS = FUSED ? Lay::FUSEDG : Lay::LOCALG;  // group region (doubles)
  static_assert(!FUSED || (kLocalGroups > 1 && kL == kLF), "fused kernel: grouped 8-element tiles");
  extern __shared__ __align__(128) double smem_cta[];
  Ctx x;
  init_ctx(x);
  x.lfs = false;
  x.qcol0 = 3 * x.w * kL;  // flux phase (8-element tiles: the unit is the tile)
  double* smem = smem_cta + x.grp * GS;  // this group's region
  // group grp of the CTA works as virtual CTA vb of a grid of vgrid
  const int64_t vb = static_cast<int64_t>(blockIdx.x) * kLocalGroups + x.grp;
  const int64_t vgrid = static_cast<int64_t>(gridDim.x) * kLocalGroups;
  x.shcap = FUSED ? Lay::LSHF : Lay::LSH;
  x.I = smem;
  x.S = smem + G::IROWS * kRS;
  x.xb = smem + Lay::ROWS * kRS + x.w * kXBUF * kXW;
  x.xb2 = x.S + (G::B - G::IROWS) * kRS + x.w * kXW;  // free during CK step 0 (Q^n fills B rows)
  x.frags = frag_table<N>();
  x.fs = kLocalGroups > 1 ? smem_cta + kLocalGroups * GS : smem + Lay::FOFF;
  x.fbar = reinterpret_cast<unsigned long long*>(smem + (FUSED ? Lay::FBAR : Lay::FOFF + Lay::FSMAX * 32));
  unsigned long long* qbar = x.fbar + 1;
  unsigned long long* fxbar = x.fbar + 2;  // fused: the flux phase's own / neighbour copies
  unsigned qph = 0, ph_o = 0, ph_n = 0;
  if constexpr (kLocalGroups > 1) {  // static fragment buffer: CK step 0, then the volume
    double* fs = const_cast<double*>(x.fs);
    for (int i = threadIdx.x; i < x.shcap * 32; i += kT * kLocalGroups) fs[i] = x.frags[i];
    __syncthreads();
  }
  if (x.tid == 0) {
    mbar_init(x.fbar, 1);
    mbar_init(qbar, 1);
    if constexpr (FUSED) {
      mbar_init(&fxbar[0], 1);
      mbar_init(&fxbar[1], 1);
    }
    if (kLocalFs && vb < prm.ntiles) stage_frags<N>(x, G::CK0_F0, G::CK0_NF < kLocalFsCap ? G::CK0_NF : kLocalFsCap);
  }
  x.sync();
  x.dt = prm.dt;
  x.scal = prm.scal;
  x.N = N;
  double* stg0 = x.S;              // trace staging blocks (S and xb are dead after CK)
  double* stg1 = x.S + Lay::FACE;
  // 3-column pattern of star-matrix row p = 3g + xk of the star-chunk role (setup.cpp
  // star_cols), packed 5 bits per column
  const int xp = 3 * (x.w / kCT) + (x.xk < kU ? x.xk : 0);
  {
    constexpr unsigned long long packed[9] = {6 | 7 << 5 | 8 << 10, 6 | 7 << 5 | 8 << 10, 6 | 7 << 5 | 8 << 10,
                                              6 | 7 << 5 | 7 << 10, 7 | 8 << 5 | 8 << 10, 6 | 8 << 5 | 8 << 10,
                                              0 | 3 << 5 | 5 << 10, 3 | 1 << 5 | 4 << 10, 5 | 4 << 5 | 2 << 10};
    unsigned long long w = 0;
#pragma unroll
    for (int i = 0; i < 9; ++i) w = (xp == i) ? packed[i] : w;
    x.q0 = static_cast<int>(w & 31);
    x.q1 = static_cast<int>((w >> 5) & 31);
    x.q2 = static_cast<int>((w >> 10) & 31);
  }
  for (int64_t it = vb; it < prm.ntiles; it += vgrid) {
    const int64_t tile = prm.tile0 + it;
    double* Qt = prm.Q + tile * B * kRS;
    YDG_PHASE(0);
    if (x.tid == 0 && (YDG_QPF & 4) == 0 && it + vgrid < prm.ntiles) {  // next tile of this CTA -> L2
      const int64_t nt = tile + vgrid;
      prefetch_l2(prm.Q + nt * B * kRS, B * kRS * sizeof(double));
      prefetch_l2(prm.star + nt * 3 * kP * 3 * kL, 3 * kP * 3 * kL * sizeof(double));
    }
    x.Qt = Qt;
    if constexpr (FUSED) {  // the previous step's flux into Q (in L2 for the staging below)
      flux_tile<N>(x, prm, tile, smem, fxbar, ph_o, ph_n);
      // the Q rows < IROWS are re-read by a bulk copy (async proxy) after the volume term
      asm volatile("fence.proxy.async.global;" ::: "memory");
      x.sync();
    }
    {  // stage Q^n of the tile in shared memory (rows of I, continuing into S): 16-byte
       // cp.async chunks, all in flight at once
      constexpr int kChunks = B * kRS / 2;
      for (int c = x.tid; c < kChunks; c += kT) {
        const int row = c / (kRS / 2), cc = 2 * (c % (kRS / 2));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(x.I + swz(row, cc))),
                     "l"(Qt + row * kRS + cc)
                     : "memory");
      }
    }
    x.star = prm.star + (tile * 3 * kP) * 3 * kL;
    const double* st = x.star + x.xe;
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int j = 0; j < 3; ++j) x.a[3 * c + j] = ld_star(st + ((c * kP + xp) * 3 + j) * kL);
    cp_async_wait_all();
    if constexpr (kLocalFs) mbar_wait(x.fbar, 0);  // CK step 0 fragments (first of two loads per tile)
    x.sync();
    YDG_PHASE(1);
    G::ck(x);  // ends with a barrier: the time integral is complete
    // traces T_F = R^FT I of the four faces -> staging -> one TMA bulk store per face;
    // they read Q^n (rows >= IROWS of I from global memory), so they precede the update
    double* gtr = prm.traces + tile * 4 * Lay::FACE;
    constexpr int F0 = G::TR23_DFMA ? 4 : (G::TR01_DFMA ? 2 : 0);
    if constexpr (G::TR01_DFMA) {
      G::trace01(x, stg0, stg1);  // faces 0 and 1: sparse DFMA
      fence_proxy_async();
      x.sync();
      if (x.tid == 0) {
        bulk_s2g(gtr, stg0, Lay::FACE * sizeof(double));
        bulk_s2g(gtr + Lay::FACE, stg1, Lay::FACE * sizeof(double));
      }
    }
    if constexpr (G::TR23_DFMA) {
      if (x.tid == 0) bulk_wait_read<0>();  // faces 0, 1 have left the staging blocks
      x.sync();
      G::trace23(x, stg0, stg1);  // faces 2 and 3: sparse DFMA
      fence_proxy_async();
      x.sync();
      if (x.tid == 0) {
        bulk_s2g(gtr + 2 * Lay::FACE, stg0, Lay::FACE * sizeof(double));
        bulk_s2g(gtr + 3 * Lay::FACE, stg1, Lay::FACE * sizeof(double));
      }
    }
#pragma unroll
    for (int F = F0; F < 4; ++F) {  // tensor-core faces
      double* stg = (F & 1) ? stg1 : stg0;
      if (F >= 2) {
        if (x.tid == 0) bulk_wait_read<1>();  // the store of face F-2 has left stg
        x.sync();
      }
      if (F == 0) G::template trace<0>(x, stg);
      else if (F == 1) G::template trace<1>(x, stg);
      else if (F == 2) G::template trace<2>(x, stg);
      else G::template trace<3>(x, stg);
      fence_proxy_async();
      x.sync();
      if (x.tid == 0) bulk_s2g(gtr + F * Lay::FACE, stg, Lay::FACE * sizeof(double));
    }
    YDG_PHASE(8);
    if (!FUSED && prm.tr_only) {  // LTS: the sub-interval traces of a coarse element, no update
      if (x.tid == 0) bulk_wait_read<0>();
      x.sync();
      continue;
    }
    if (x.tid == 0) bulk_wait_read<0>();
    x.sync();  // the staging blocks overlap the X buffers of the volume term
    if (x.tid == 0) {  // rows < IROWS of Q^n -> S (free now) for the volume's update
      mbar_expect_tx(qbar, G::IROWS * kRS * sizeof(double));
      bulk_g2s(x.S, Qt, G::IROWS * kRS * sizeof(double), qbar);
    }
    if constexpr ((YDG_QPF & 2) != 0)
      if (x.tid == 32) prefetch_l2(Qt + G::IROWS * kRS, (B - G::IROWS) * kRS * sizeof(double));
    if constexpr ((YDG_QPF & 4) != 0)  // bit 4: the next tile's Q^n and star matrices -> L2 now
      if (x.tid == 64 && it + vgrid < prm.ntiles) {
        const int64_t nt = tile + vgrid;
        prefetch_l2(prm.Q + nt * B * kRS, B * kRS * sizeof(double));
        prefetch_l2(prm.star + nt * 3 * kP * 3 * kL, 3 * kP * 3 * kL * sizeof(double));
      }
    YDG_PHASE(9);
    {
      double acc[G::QMT][kU][2];
      zero_acc(acc);
      if constexpr (kLocalFs) mbar_wait(x.fbar, 1);  // volume fragments (staged after CK step 0)
      // YDG_VOL_QEARLY: the Q update's first global rows loaded before the volume product
      double2 vpre[2][kU];
      if constexpr (YDG_VOL_QEARLY) G::add_volume_pre(x, Qt, vpre);
      G::volume(x, acc);
      YDG_PHASE(10);
      mbar_wait(qbar, qph);
      qph ^= 1;
      G::add_volume(x, Qt, acc, x.S, YDG_VOL_QEARLY ? vpre : nullptr);
    }
    x.sync();  // before the next tile overwrites the shared regions
    if (kLocalFs && x.tid == 0 && it + vgrid < prm.ntiles)
      stage_frags<N>(x, G::CK0_F0, G::CK0_NF < kLocalFsCap ? G::CK0_NF : kLocalFsCap);
    YDG_PHASE(11);
#ifdef YDG_PHASES
    if (x.tid == 0 && vb == 0 && it >= 2 * vgrid && it < 6 * vgrid) {
      printf("PH tile %lld: stage %lld ck %lld %lld %lld %lld %lld %lld traces %lld wait %lld vol %lld addq %lld total %lld\n",
             (long long)it, ph_t[1] - ph_t[0], ph_t[2] - ph_t[1], ph_t[3] - ph_t[2], ph_t[4] - ph_t[3],
             ph_t[5] - ph_t[4], ph_t[6] - ph_t[5], ph_t[7] - ph_t[6], ph_t[8] - ph_t[7], ph_t[9] - ph_t[8],
             ph_t[10] - ph_t[9], ph_t[11] - ph_t[10], ph_t[11] - ph_t[0]);
    }
#endif
  }
  if (x.tid == 0) bulk_wait_all();
}

template <int N>
__global__ void __launch_bounds__(kT * kLocalGroups, kLocalGroups == 1 ? kDmCtasPerSm : 1)
    dm_local(const __grid_constant__ StepParams<double> prm) {
  local_body<N, false>(prm);
}

// Fused step kernel: per tile, the flux of the previous step (own and neighbour traces from
// prm.traces_in) added to Q, then CK, time integral, traces (-> prm.traces) and
// the volume term of this step.  The tile's Q is read from HBM once and written
// once per step; the flux phases' memory latency overlaps the other groups' tensor-core work.
template <int N>
__global__ void __launch_bounds__(kT * kLocalGroups, 1) dm_fused(const __grid_constant__ StepParams<double> prm) {
  if constexpr (kLocalGroups > 1 && kL == kLF) local_body<N, true>(prm);
}

// Flux kernel: local and neighbour flux with one lift per face:
//   Q += sum_i R^i ( T_i A+_i^T + (f^h_i T^nb_(j_i)) A-_i^T ).
// Per (tile, face) item: one TMA bulk copy of the tile's own face block (buffer O) and one
// per lane of the neighbour's face block (buffers N0/N1: the next face's copies are in
// flight while this one computes); f^h rotates the neighbour column in place, thread
// (e, m) builds the Godunov flux of row m from T and Z (godunov_flux), writing Y (rows
// [m][288]), and the warp lifts its own columns of Y with DMMAs into Q.
template <int N>
__global__ void __launch_bounds__(kTF * kFluxGroups, kFluxGroups == 1 ? kFluxCtas : 1)
    dm_flux(const __grid_constant__ StepParams<double> prm) {
  using G = DG<N>;
  using Lay = Layout<N>;
  constexpr int B = G::B, Bt = G::Bt, TS = G::TS, FACE = Lay::FACE, FACEF = Lay::FACEF;
  constexpr int FCN = kFaceCoeffs * kLF;  // factored flux solvers of one (tile, face, half)
  extern __shared__ __align__(128) double smem_cta[];
  // group grp (3 warps) of the CTA works as one virtual CTA vb of a grid of vgrid
  const int grp = threadIdx.x / kTF, tid = threadIdx.x % kTF;
  const int64_t vb = static_cast<int64_t>(blockIdx.x) * kFluxGroups + grp;
  const int64_t vgrid = static_cast<int64_t>(gridDim.x) * kFluxGroups;
  double* smem = smem_cta + grp * Lay::FLUXG;
  auto gsync = [&]() {
    if constexpr (kFluxGroups == 1) __syncthreads();
    else asm volatile("bar.sync %0, %1;" ::"r"(grp + 1), "n"(kTF) : "memory");
  };
  double* O = smem;                    // own face block [lane][TS] of the CTA's 8 elements
  double* NB = smem + FACEF;           // [lane][TS] neighbour face blocks
  double* Y0 = smem + 2 * FACEF;       // [2][Bt][72]: rotated neighbour rows, then the flux
  double* FC = Y0 + 2 * Bt * kRSF;     // [12][8] flux coefficients of the current item
  int32_t* NBX = reinterpret_cast<int32_t*>(FC + FCN);  // [8] neighbour slots of the next item
  int8_t* JH = reinterpret_cast<int8_t*>(NBX + kLF);    // [16] j | h << 2 of the current (tile, face)
  int8_t* JHX = JH + kJH;                               // [16] of the next item's (tile, face)
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(JHX + kJH);  // own, nb
  Ctx x;
  x.shcap = 0;  // (the local kernel's shared fragment slots)
  x.lfs = true;
  x.lane = tid & 31;
  x.w = tid >> 5;
  x.col0 = 3 * x.w * kLF;
  x.sh4 = 8 * (x.lane & 3);
  x.sh8 = 8 * (x.lane >> 2);
  x.frags = frag_table<N>();
  if constexpr (kFluxFs) {  // the lift's A fragments, once per CTA
    double* fs = smem_cta + kFluxGroups * Lay::FLUXG;
    for (int i = threadIdx.x; i < G::LIFT_NF * 32; i += kTF * kFluxGroups) fs[i] = x.frags[G::LIFT_F0 * 32 + i];
    x.fs = fs;
    __syncthreads();
  }
  const int64_t nitems = prm.ntiles * kHalves;  // (tile, half) work units
  if (vb >= nitems) return;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
  }
  gsync();
  // Items k = (unit, face) in this CTA's order, unit = (tile, half); item k's "own" copy
  // (thread 0) brings the unit's face block, its flux coefficients and j|h, and the
  // neighbour slots and j|h of item k+1, so no global load sits on the per-face path.
  auto issue_own = [&](int64_t u, int F, int64_t nu, int nF, bool next) {
    const int64_t tile = prm.tile0 + u / kHalves, half = u % kHalves;
    const int64_t ntile = prm.tile0 + nu / kHalves, nhalf = nu % kHalves;
    const int64_t item = tile * 4 + F, nitem = ntile * 4 + nF;
    mbar_expect_tx(&bar[0], (FACEF + FCN) * sizeof(double) + kJH + (next ? kLF * 4 + kJH : 0));
    bulk_g2s(O, prm.traces + item * FACE + half * FACEF, FACEF * sizeof(double), &bar[0]);
#pragma unroll
    for (int k = 0; k < kFaceCoeffs; ++k)
      bulk_g2s(FC + k * kLF, prm.aplus + (item * kFaceCoeffs + k) * kL + half * kLF, kLF * sizeof(double), &bar[0]);
    bulk_g2s(JH, prm.jh + item * kJH, kJH, &bar[0]);
    if (next) {
      bulk_g2s(NBX, prm.nb + nitem * kL + nhalf * kLF, kLF * sizeof(int32_t), &bar[0]);
      bulk_g2s(JHX, prm.jh + nitem * kJH, kJH, &bar[0]);
    }
  };
  auto issue_nb = [&](const int32_t* nbs, const int8_t* jhs) {  // thread 0; jhs = this half's 8
    mbar_expect_tx(&bar[1], FACEF * sizeof(double));
#pragma unroll
    for (int e = 0; e < kLF; ++e) {
      const int64_t nbe = nbs[e];
      bulk_g2s(NB + e * TS, prm.traces + ((nbe / kL) * 4 + (jhs[e] & 3)) * FACE + (nbe % kL) * TS,
               TS * sizeof(double), &bar[1]);
    }
  };
  {
    const int64_t u0 = vb;
    if (tid == 0) {
      const int64_t tile = prm.tile0 + u0 / kHalves, half = u0 % kHalves;
      int32_t nbs[kLF];
      int8_t jhs[kLF];
#pragma unroll
      for (int e = 0; e < kLF; ++e) {
        nbs[e] = prm.nb[tile * 4 * kL + half * kLF + e];
        jhs[e] = prm.jh[tile * 4 * kJH + half * kLF + e];
      }
      issue_nb(nbs, jhs);
      issue_own(u0, 0, u0, 1, true);
    }
  }
  unsigned ph_o = 0, ph_n = 0;
  // thread roles: rotation (element re, column rp) for threads < 72; Godunov rows
  // m = rp + 12 i of element re
  const int re = tid % kLF, rp = tid / kLF;
  // YDG_FLUX_LATE_OWN: the rotation takes h from a register (read from the previous item's
  // j|h copy), so the wait for the own copy moves behind the rotation
  int hcur = 0;
  if constexpr (kFluxLateOwn) hcur = prm.jh[(prm.tile0 + vb / kHalves) * 4 * kJH + (vb % kHalves) * kLF + re] >> 2;
  for (int64_t u = vb; u < nitems; u += vgrid) {
    const int64_t tile = prm.tile0 + u / kHalves, half = u % kHalves;
    x.qcol0 = 3 * x.w * kL + half * kLF;
    const bool more = u + vgrid < nitems;
#pragma unroll
    for (int F = 0; F < 4; ++F) {
      // Y buffer F & 1: last read by the paired lift of faces F-2, F-1 (followed by a barrier)
      double* Y = Y0 + (F & 1) * Bt * kRSF;
      const bool has_next = F < 3 || more;
      double* Qt = prm.Q + tile * B * kRS;
      double2 qn[2][kU];
      // YDG_FLUX_QEARLY: the lift's first Q rows are loaded early, their L2 latency
      // overlapping the Godunov flux (1) or also the waits and the rotation (2)
      if (kFluxQEarly == 2 && (F & 1)) G::lift2_pre(x, Qt, qn);
      if constexpr (!kFluxLateOwn) {
        mbar_wait(&bar[0], ph_o);  // own block, coefficients, j|h of this item; slots of the next
        ph_o ^= 1;
      }
      mbar_wait(&bar[1], ph_n);  // neighbour blocks of this item
      ph_n ^= 1;
      if (tid < kP * kLF) {  // z = f^h t on column rp of element re's neighbour block -> Y
        const int h = kFluxLateOwn ? hcur : JH[half * kLF + re] >> 2;
        const double* zc = NB + re * TS + rp;
        double t[Bt];
#pragma unroll
        for (int n = 0; n < Bt; ++n) t[n] = zc[n * kP];
        G::rotf(h, t, Y, rp * kLF + re);
      }
      if constexpr (kFluxLateOwn) {
        mbar_wait(&bar[0], ph_o);  // own block, coefficients of this item; slots, j|h of the next
        ph_o ^= 1;
        if (has_next) hcur = JHX[(F < 3 ? half : (u + vgrid) % kHalves) * kLF + re] >> 2;
      }
      double fc[kFaceCoeffs];
#pragma unroll
      for (int k = 0; k < kFaceCoeffs; ++k) fc[k] = FC[k * kLF + re];
      gsync();  // rotated rows visible; every read of NB (and of NBX, JHX) done
      if (tid == 0 && has_next) {
        const int nhalf = F < 3 ? half : (u + vgrid) % kHalves;
        issue_nb(NBX, JHX + nhalf * kLF);
      } else if (tid == 32 && F == kFluxQpfFace && more) {  // next unit's Q -> L2
        prefetch_l2(prm.Q + (prm.tile0 + (u + vgrid) / kHalves) * B * kRS, B * kRS * sizeof(double));
      }
      if constexpr (kFluxPf != 0) {  // the next unit's face blocks -> L2, half a unit ahead
        if (F == kFluxPfFace && more && tid >= 64) {
          const int64_t nu = u + vgrid, ntile = prm.tile0 + nu / kHalves, nhalf = nu % kHalves;
          const int k = tid - 64, f = k / kLF, e = k % kLF;  // 32 threads: (face, element)
          if (kFluxPf & 1) {  // neighbour blocks
            const int64_t slot = (ntile * 4 + f) * kL + nhalf * kLF + e;
            const int64_t nbe = prm.nb[slot];
            const int jn = prm.jh[(ntile * 4 + f) * kJH + nhalf * kLF + e] & 3;
            prefetch_l2(prm.traces + ((nbe / kL) * 4 + jn) * FACE + (nbe % kL) * TS, TS * sizeof(double));
          }
          if ((kFluxPf & 2) && e == 0)  // own face blocks
            prefetch_l2(prm.traces + (ntile * 4 + f) * FACE + nhalf * FACEF, FACEF * sizeof(double));
        }
      }
      if (kFluxQEarly == 1 && (F & 1)) G::lift2_pre(x, Qt, qn);
      {  // Godunov flux of rows m = rp, rp + 12, ... of element re, in place in Y
        const double* T = O + re * TS;
#pragma unroll
        for (int i = 0; i < (Bt + kTF / kLF - 1) / (kTF / kLF); ++i) {
          const int m = rp + (kTF / kLF) * i;
          if (m >= Bt) break;
          double z[kP], y[kP];
#pragma unroll
          for (int q = 0; q < kP; ++q) z[q] = Y[swzf(m, q * kLF + re)];
          godunov_flux(T + m * kP, z, fc, y);
#pragma unroll
          for (int q = 0; q < kP; ++q) Y[swzf(m, q * kLF + re)] = y[q];
        }
      }
      gsync();  // every read of O, FC, JH done; Y complete
      if (tid == 0 && has_next) {  // item k+1's own copy (and item k+2's slots)
        const int64_t nu = F < 3 ? u : u + vgrid;
        const int nF = F < 3 ? F + 1 : 0;
        const bool nn = nF < 3 || nu + vgrid < nitems;
        issue_own(nu, nF, nF < 3 ? nu : nu + vgrid, nF < 3 ? nF + 1 : 0, nn);
      }
      // lift and Q update per pair of faces (both Y buffers), two m-tiles at a time; the
      // unit's Q stays in L2 across its two updates.  The next pair's rotation rewrites the
      // Y buffers: a barrier after the lift.
      if (F & 1) {
        if (kFluxQEarly == 0) G::lift2_pre(x, Qt, qn);
        if (F == 1) G::template lift2<0>(x, Y0, Y0 + Bt * kRSF, Qt, qn);
        else G::template lift2<1>(x, Y0, Y0 + Bt * kRSF, Qt, qn);
        gsync();
      }
    }
  }
}

// Flux phase of the fused kernel for one 8-element tile (= one flux unit): the per-face work
// of dm_flux -- own face block, flux coefficients and j|h by one bulk copy group, the eight
// neighbour face blocks by another (the next face's copies in flight while this face
// computes), f^h rotation, Godunov flux, paired lift + Q update -- on this group's region
// (the local phase's buffers are dead here).  Traces come from prm.traces_in.
template <int N>
__device__ __forceinline__ void flux_tile(Ctx& x, const StepParams<double>& prm, int64_t tile, double* smem,
                                          unsigned long long* bar, unsigned& ph_o, unsigned& ph_n) {
  using G = DG<N>;
  using Lay = Layout<N>;
  constexpr int B = G::B, Bt = G::Bt, TS = G::TS, FACE = Lay::FACE, FACEF = Lay::FACEF;
  constexpr int FCN = kFaceCoeffs * kLF;
  const int tid = x.tid;
  double* O = smem;
  double* NB = smem + FACEF;
  double* Y0 = smem + 2 * FACEF;
  double* FC = Y0 + 2 * Bt * kRSF;
  int32_t* NBX = reinterpret_cast<int32_t*>(FC + FCN);
  int8_t* JH = reinterpret_cast<int8_t*>(NBX + kLF);
  int8_t* JHX = JH + kJH;
  const double* tin = prm.traces_in;
  auto issue_own = [&](int F, bool next) {  // thread 0: item (tile, F); slots, j|h of (tile, F + 1)
    const int64_t item = tile * 4 + F;
    mbar_expect_tx(&bar[0], (FACEF + FCN) * sizeof(double) + kJH + (next ? kLF * 4 + kJH : 0));
    bulk_g2s(O, tin + item * FACE, FACEF * sizeof(double), &bar[0]);
#pragma unroll
    for (int k = 0; k < kFaceCoeffs; ++k)
      bulk_g2s(FC + k * kLF, prm.aplus + (item * kFaceCoeffs + k) * kL, kLF * sizeof(double), &bar[0]);
    bulk_g2s(JH, prm.jh + item * kJH, kJH, &bar[0]);
    if (next) {
      bulk_g2s(NBX, prm.nb + (item + 1) * kL, kLF * 4, &bar[0]);
      bulk_g2s(JHX, prm.jh + (item + 1) * kJH, kJH, &bar[0]);
    }
  };
  auto issue_nb = [&](const int32_t* nbs, const int8_t* jhs) {  // thread 0
    mbar_expect_tx(&bar[1], FACEF * sizeof(double));
#pragma unroll
    for (int e = 0; e < kLF; ++e) {
      const int64_t nbe = nbs[e];
      bulk_g2s(NB + e * TS, tin + ((nbe / kL) * 4 + (jhs[e] & 3)) * FACE + (nbe % kL) * TS, TS * sizeof(double),
               &bar[1]);
    }
  };
  if (tid == 0) {
    fence_proxy_async();  // the local phase's generic accesses to the region, then the copies
    int32_t nbs[kLF];
    int8_t jhs[kLF];
#pragma unroll
    for (int e = 0; e < kLF; ++e) {
      nbs[e] = prm.nb[tile * 4 * kL + e];
      jhs[e] = prm.jh[tile * 4 * kJH + e];
    }
    issue_nb(nbs, jhs);
    issue_own(0, true);
  } else if (tid == 32) {
    prefetch_l2(prm.Q + tile * B * kRS, B * kRS * sizeof(double));  // the lifts' read-modify-write
  }
  const int re = tid % kLF, rp = tid / kLF;
  double* Qt = prm.Q + tile * B * kRS;
#pragma unroll
  for (int F = 0; F < 4; ++F) {
    double* Y = Y0 + (F & 1) * Bt * kRSF;
    mbar_wait(&bar[0], ph_o);  // own block, coefficients, j|h of this face; slots of the next
    ph_o ^= 1;
    mbar_wait(&bar[1], ph_n);  // neighbour blocks of this face
    ph_n ^= 1;
    if (tid < kP * kLF) {  // z = f^h t on column rp of element re's neighbour block -> Y
      const int h = JH[re] >> 2;
      const double* zc = NB + re * TS + rp;
      double t[Bt];
#pragma unroll
      for (int n = 0; n < Bt; ++n) t[n] = zc[n * kP];
      G::rotf(h, t, Y, rp * kLF + re);
    }
    double fc[kFaceCoeffs];
#pragma unroll
    for (int k = 0; k < kFaceCoeffs; ++k) fc[k] = FC[k * kLF + re];
    x.sync();  // rotated rows visible; every read of NB (and of NBX, JHX) done
    if (tid == 0 && F < 3) issue_nb(NBX, JHX);
    {  // Godunov flux of rows m = rp, rp + 12, ... of element re, in place in Y
      const double* T = O + re * TS;
#pragma unroll
      for (int i = 0; i < (Bt + kTF / kLF - 1) / (kTF / kLF); ++i) {
        const int m = rp + (kTF / kLF) * i;
        if (m >= Bt) break;
        double z[kP], y[kP];
#pragma unroll
        for (int q = 0; q < kP; ++q) z[q] = Y[swzf(m, q * kLF + re)];
        godunov_flux(T + m * kP, z, fc, y);
#pragma unroll
        for (int q = 0; q < kP; ++q) Y[swzf(m, q * kLF + re)] = y[q];
      }
    }
    x.sync();  // every read of O, FC, JH done; Y complete
    if (tid == 0 && F < 3) issue_own(F + 1, F + 1 < 3);
    if (F & 1) {  // lift of the face pair + Q update; the pair's Y buffers are reused after
      double2 qn[2][kU];
      G::lift2_pre(x, Qt, qn);
      if (F == 1) G::template lift2<0>(x, Y0, Y0 + Bt * kRSF, Qt, qn);
      else G::template lift2<1>(x, Y0, Y0 + Bt * kRSF, Qt, qn);
      if (F == 1) x.sync();
    }
  }
}

}  // namespace dm
}  // namespace ydg
