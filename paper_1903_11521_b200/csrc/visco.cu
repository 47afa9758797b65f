// Viscoelastic (P = 27, three mechanisms) local kernel on FP64 tensor cores, orders N <= 4.
//
// One persistent CTA per SM walks tiles of TE = 8 consecutive elements and runs the whole
// element-local part of one ADER-DG step (SURVEY §8 rows A3-A6 with A9; P:1312-1341 and the
// source term of reading R14):
//
//   D^0 = Q;  D^{d+1} = dt/(d+1) (sum_c Ktilde^c D^d A*^cT + D^d E^T);  I = dt sum_d D^d / (d+1)
//   Q += sum_c Khat^c I A*^cT + I E^T + sum_i R^i (R^iT I) A+_i^T;   traces T_i = R^iT I (q < 9)
//
// Data columns are (quantity p, element e) -> p * 8 + e, so one 8-column DMMA B operand is one
// quantity of the tile's 8 elements.  Warp w owns the three quantities of group g(w); every
// product with a global matrix M (Ktilde^c, Khat^c, R^i, R^iT) runs as m8n8k4 tiles over the
// generated, zero-block-free tile lists of generated/ydg_visco.cuh, with the warp's B fragments
// computed straight into registers from shared memory (the star / flux-solver right-multiply
// of 4 rows at a time: X^c = D A*^cT, Y_i = T_i A+_iT) -- no intermediate ever leaves the SM.
// The time integral I lives in the accumulator layout in registers during the recursion.
#include <cuda_runtime.h>

#include <cstdint>

#include "generic.h"
#include "generated/ydg_visco.cuh"

namespace ydg {
namespace visco {

constexpr int P = 27, TE = 8, W = 9, NTH = W * 32;
constexpr int SD = P * TE + 1;   // D / I row stride in doubles (odd: consecutive rows on distinct banks)
constexpr int TS = 9 * TE + 12;  // trace row stride


// measured (c3, vm_local): 41.63 -> 40.78 ms (YDG_VCOMB) -> 39.60 ms (+ YDG_VQB)
#ifndef YDG_VCOMB
#define YDG_VCOMB 1
#endif
#ifndef YDG_VQB
#define YDG_VQB 1
#endif
// Bulk L2 prefetch of [p, p + bytes), widened to 16-byte alignment (the instruction's rule).
__device__ __forceinline__ void l2_prefetch(const void* p, int64_t bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p), a0 = a & ~uintptr_t(15);
  const int n = static_cast<int>((a + bytes - a0 + 15) & ~int64_t(15));
  if (bytes > 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"(n) : "memory");
}

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}

__device__ __forceinline__ void st2(double* p, double a, double b) {  // (odd row strides: 8-byte aligned only)
  p[0] = a;
  p[1] = b;
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// Quantity group of warp w (quantities 3g..3g+2): the velocity group (no source term) and the
// source-heavy stress groups go to the sub-partitions that hold two warps, not three.
__device__ __forceinline__ int group_of(int w) { return w == 0 ? 3 : w == 1 ? 2 : w == 2 ? 0 : w == 3 ? 1 : w; }

template <int N>
struct Ctx {
  using V = VT<N>;
  const double* D;     // shared: D^d (recursion) / I (volume, traces) [BR][SD]
  const double* TR;    // shared: traces [4][BtR][TS]
  const double* FR;    // shared: A fragments [NFRAG][32]
  const double* ap;    // global: A+- of the lane's element [face][p][9]
  int lane, k, e, p0, q;
  double a[3][9];      // flux-solver coefficients of the current face
  double b[2][3];      // lift B fragments (double-buffered one k-set ahead)
  double b1[2];

  __device__ __forceinline__ void ib(int buf, int ks) { b1[buf] = D[(4 * ks + k) * SD + q * TE + e]; }
  __device__ __forceinline__ void mma1(double (&acc)[2], int f, int buf) { dmma(acc, FR[f * 32 + lane], b1[buf]); }
  __device__ __forceinline__ void mma(double (&acc)[3][2], int f, int buf) {
    const double af = FR[f * 32 + lane];
    dmma(acc[0], af, b[buf][0]);
    dmma(acc[1], af, b[buf][1]);
    dmma(acc[2], af, b[buf][2]);
  }
  __device__ __forceinline__ void acoef(int i) {
#pragma unroll
    for (int u = 0; u < 3; ++u)
#pragma unroll
      for (int j = 0; j < 9; ++j) a[u][j] = ap[(i * P + p0 + u) * 9 + j];
    if (i < 3)  // the next face's rows -> L1 (three 72-byte rows per lane)
#pragma unroll
      for (int u = 0; u < 3; ++u)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(ap + ((i + 1) * P + p0 + u) * 9));
  }
  __device__ __forceinline__ void ychunk(int buf, int i, int ks) {
    const double* r = TR + (i * V::BtR + 4 * ks + k) * TS + e;
    double t[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) t[j] = r[j * TE];
#pragma unroll
    for (int u = 0; u < 3; ++u) {  // three short chains (DFMA latency), summed
      const double y0 = fma(a[u][2], t[2], fma(a[u][1], t[1], a[u][0] * t[0]));
      const double y1 = fma(a[u][5], t[5], fma(a[u][4], t[4], a[u][3] * t[3]));
      const double y2 = fma(a[u][8], t[8], fma(a[u][7], t[7], a[u][6] * t[6]));
      b[buf][u] = y0 + y1 + y2;
    }
  }
};

template <int N, class X, int M>
__device__ __forceinline__ void ck(X& x, double (&a)[3][M][2]) {
  if constexpr (N == 1) vck1(x, a);
  else if constexpr (N == 2) vck2(x, a);
  else if constexpr (N == 3) vck3(x, a);
  else vck4(x, a);
}
template <int N, class X, int M>
__device__ __forceinline__ void vol(X& x, double (&a)[3][M][2]) {
  if constexpr (N == 1) vvol1(x, a);
  else if constexpr (N == 2) vvol2(x, a);
  else if constexpr (N == 3) vvol3(x, a);
  else vvol4(x, a);
}
template <int N, class X, int M>
__device__ __forceinline__ void lift(X& x, double (&a)[M][3][2]) {
  if constexpr (N == 1) vlift1(x, a);
  else if constexpr (N == 2) vlift2(x, a);
  else if constexpr (N == 3) vlift3(x, a);
  else vlift4(x, a);
}
template <int N, class X, int M>
__device__ __forceinline__ void traces(X& x, double (&t)[4][M][2]) {
  if constexpr (N == 1) vtr1(x, t);
  else if constexpr (N == 2) vtr2(x, t);
  else if constexpr (N == 3) vtr3(x, t);
  else vtr4(x, t);
}

template <int M, class F>
__device__ __forceinline__ void rows_of(F words, int ar, int (&rows)[M]) {
#pragma unroll
  for (int mt = 0; mt < M; ++mt) {
    const int r = static_cast<int>((words(mt) >> (8 * ar)) & 0xffull);
    rows[mt] = r == 0xff ? -1 : r;
  }
}

// Star / source combination of one (row r, element e) of the left-first products
// Z^c_t = M^c X_t (c = 0..2, t = the 9 elastic quantities; Z[c][r][t][e] in shared memory):
//   out_p = sum_c sum_t A*^c[p][t] Z^c_t + sum_j E[p][j] X_j        (reading R14 source)
// Every non-velocity row reads the velocity columns (VU, VV, VW) in order, the velocity rows
// the stresses (SXX SXY SXZ) (SXY SYY SYZ) (SXZ SYZ SZZ) (setup.cpp star_cols, P = 27); the
// source couples normal stresses to the 9 normal memory variables, shear stresses to 3, and
// each memory variable to itself.  emit(p, value) receives every output exactly once.
constexpr int ZS = 9 * TE + 1;  // Z row stride (odd)
constexpr int CSS = 10;      // star coefficients per (element, row): [c][t], padded
constexpr int CSE = P * CSS;
constexpr int CEE = 57;      // source coefficients per element (54 used; odd stride: no bank conflicts)

template <int B>
__device__ __forceinline__ double star_row(int p, const double* cs, const double (&z)[3][3]) {
  const double* c = cs + p * CSS;  // [c*3+t]; warp-uniform addresses (broadcast)
  const double s0 = fma(c[2], z[0][2], fma(c[1], z[0][1], c[0] * z[0][0]));
  const double s1 = fma(c[5], z[1][2], fma(c[4], z[1][1], c[3] * z[1][0]));
  const double s2 = fma(c[8], z[2][2], fma(c[7], z[2][1], c[6] * z[2][0]));
  return (s0 + s1) + s2;
}
__device__ __forceinline__ double source_row(int p, const double* ce, const double (&m)[18]) {
  double sr = 0.0;
  if (p < 3) {
#if YDG_VCOMB
    double s3[3];  // three independent chains (one per mechanism): no 9-deep FMA dependency
#pragma unroll
    for (int l = 0; l < 3; ++l)
      s3[l] = fma(ce[p * 9 + 3 * l + 2], m[6 * l + 2], fma(ce[p * 9 + 3 * l + 1], m[6 * l + 1], ce[p * 9 + 3 * l] * m[6 * l]));
    sr = (s3[0] + s3[1]) + s3[2];
#else
#pragma unroll
    for (int l = 0; l < 3; ++l)
#pragma unroll
      for (int t = 0; t < 3; ++t) sr = fma(ce[p * 9 + 3 * l + t], m[6 * l + t], sr);
#endif
  } else if (p < 6) {
#pragma unroll
    for (int l = 0; l < 3; ++l) sr = fma(ce[27 + (p - 3) * 3 + l], m[6 * l + p], sr);
  } else if (p >= 9) {
    sr = ce[36 + p - 9] * m[p - 9];
  }
  return sr;
}

// VEL_FIRST: the velocity rows (stress columns) before the others, with every Z value of the
// thread loaded up front -- the volume writes its result into the thread's own Z slots.
template <int B, bool VEL_FIRST, class Emit>
__device__ __forceinline__ void combine(const double* zr, const double* xr, const double* cs, const double* ce,
                                        const double (&wr)[3], Emit emit) {
  constexpr int cols[3][3] = {{0, 3, 5}, {3, 1, 4}, {5, 4, 2}};
  double m[18], zv[3][3];
#pragma unroll
  for (int j = 0; j < 18; ++j) m[j] = xr[(9 + j) * TE];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int t = 0; t < 3; ++t) zv[c][t] = zr[c * B * ZS + (6 + t) * TE];
  auto vel_rows = [&]() {
    double zs[3][6];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int t = 0; t < 6; ++t) zs[c][t] = zr[c * B * ZS + t * TE];
    double v[3];
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      double z[3][3];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int t = 0; t < 3; ++t) z[c][t] = zs[c][cols[u][t]];
      v[u] = star_row<B>(6 + u, cs, z);
    }
#pragma unroll
    for (int u = 0; u < 3; ++u) emit(6 + u, v[u]);
  };
#if YDG_VCOMB
  // YDG_VCOMB: every coefficient load of a batch before its stores (the emits write shared
  // memory, which the compiler must assume aliases the coefficient rows): batch A = the
  // velocity and stress rows, batch B = the memory variables, each a set of independent
  // chains
  {
    double zs[3][6];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int t = 0; t < 6; ++t) zs[c][t] = zr[c * B * ZS + t * TE];
    double oa[9];
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      double z[3][3];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int t = 0; t < 3; ++t) z[c][t] = zs[c][cols[u][t]];
      oa[6 + u] = star_row<B>(6 + u, cs, z);
    }
#pragma unroll
    for (int p = 0; p < 6; ++p) oa[p] = star_row<B>(p, cs, zv) + source_row(p, ce, m);
#pragma unroll
    for (int p = 0; p < 9; ++p) emit(p, oa[p]);
  }
  {
    double base[6], ob[18];
#pragma unroll
    for (int p = 9; p < 15; ++p) base[p - 9] = star_row<B>(p, cs, zv);
#pragma unroll
    for (int p = 9; p < P; ++p)
      ob[p - 9] = (p < 15 ? base[p - 9] : wr[(p - 9) / 6] * base[(p - 9) % 6]) + source_row(p, ce, m);
#pragma unroll
    for (int p = 9; p < P; ++p) emit(p, ob[p - 9]);
  }
  return;
#endif
  if (VEL_FIRST) vel_rows();
  // memory variables: the star rows of mechanism l are omega_l / omega_0 times those of
  // mechanism 0 (A^d rows -omega_l eps(v); checked at upload), so 6 rows are contracted
  double base[6];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    if (p >= 6 && p < 9) continue;
    double sv;
    if (p < 15) {
      sv = star_row<B>(p, cs, zv);
      if (p >= 9) base[p - 9] = sv;
    } else {
      sv = wr[(p - 9) / 6] * base[(p - 9) % 6];
    }
    emit(p, sv + source_row(p, ce, m));
  }
  if (!VEL_FIRST) vel_rows();
}

template <int N>
constexpr int dsz() {  // D buffer (also holds the traces after the recursion); even: 16-byte alignment
  return ((VT<N>::BR * SD > 4 * VT<N>::BtR * TS ? VT<N>::BR * SD : 4 * VT<N>::BtR * TS) + 1) & ~1;
}
template <int N>
constexpr int zsize() { return (3 * VT<N>::B * ZS + 1) & ~1; }
template <int N>
constexpr size_t smem_bytes() {
  return (static_cast<size_t>(dsz<N>()) + zsize<N>() + VT<N>::NFRAG * 32 + TE * (CSE + CEE)) * sizeof(double);
}

template <int N>
__global__ void __launch_bounds__(NTH, 1) vm_local(const GenParams prm) {
  using V = VT<N>;
  constexpr int B = V::B, Bt = V::Bt, KB = (B + 3) / 4;
  extern __shared__ __align__(16) double sm[];
  double* D = sm;                   // D^d, then I; after the traces: traces [4][BtR][TS], Q staging
  double* TR = D;
  double* Z = D + dsz<N>();         // left-first products Z^c_t [3][B][ZS]; after the volume: its result
  double* FR = Z + zsize<N>();
  double* CS = FR + V::NFRAG * 32;  // the tile's star rows [e][p][c*3+t] and sources [e][56]
  double* CE = CS + TE * CSE;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = group_of(w), p0 = 3 * g;
  {
    const double* f = vfrag<N>();
    for (int i = tid; i < V::NFRAG * 32; i += NTH) FR[i] = f[i];
    for (int i = tid; i < dsz<N>(); i += NTH) D[i] = 0.0;  // padding rows stay zero
  }
  Ctx<N> x;
  x.D = D;
  x.TR = TR;
  x.FR = FR;
  x.lane = lane;
  x.k = lane & 3;
  x.e = lane >> 2;
  x.p0 = p0;
  x.q = w;  // left-first / trace column of this warp (elastic quantity w < 9)
  const int ar = lane >> 2, ae = 2 * (lane & 3);  // accumulator row slot / first element
  // combination thread (row cr, element cel): warps 0..7 take rows 0..31 of element w (the
  // element's coefficients are warp-uniform: broadcast loads), warp 8 the rows >= 32
  const int cr = w < TE ? lane : 32 + lane % (B > 32 ? B - 32 : 1);
  const int cel = w < TE ? w : lane / (B > 32 ? B - 32 : 1);
  const bool comb = w < TE ? lane < B : (B > 32 && lane < TE * (B - 32));

  const int64_t ntiles = (prm.n + TE - 1) / TE;
  // Q^n of a tile -> Z (element-major, as in HBM) by cp.async: the first tile's now, each
  // next tile's while the current one is lifted (Z is free then)
  auto issue_q = [&](int64_t t) {
    const int64_t n0 = prm.e0 + t * TE;
    const int nl = static_cast<int>(prm.e0 + prm.n - n0 < TE ? prm.e0 + prm.n - n0 : TE);
    const double* Qt = prm.Q + n0 * P * B;  // n0 % 8 == 0: 16-byte aligned
    const int n = nl * P * B;
    for (int i = tid; i < n / 2; i += NTH) cp_async16(Z + 2 * i, Qt + 2 * i);
    if ((n & 1) && tid == 0) cp_async8(Z + n - 1, Qt + n - 1);
  };
  if (blockIdx.x < ntiles) issue_q(blockIdx.x);
  // the tile's star rows [e][c][p][t] -> CS [e][p][c*3+t] and compact source rows -> CE,
  // by cp.async (asynchronously for the next tile, once the current one's volume is done)
  auto coeffs = [&](int64_t t, bool async) {
    const int64_t n0 = prm.e0 + t * TE;
    const int nl = static_cast<int>(prm.e0 + prm.n - n0 < TE ? prm.e0 + prm.n - n0 : TE);
    const double* St = prm.star + n0 * 3 * P * 3;
    const double* Et = prm.src + n0 * P * 9;
    for (int i = tid; i < TE * 3 * P * 3; i += NTH) {
      const int ee = i / (3 * P * 3), r = i - ee * 3 * P * 3, c = r / (P * 3), pt = r - c * P * 3;
      double* d = CS + ee * CSE + (pt / 3) * CSS + c * 3 + pt % 3;
      if (ee >= nl) *d = 0.0;
      else if (async) cp_async8(d, St + i);
      else *d = St[i];
    }
    for (int i = tid; i < TE * CEE; i += NTH) {
      const int ee = i / CEE, j = i - ee * CEE;
      const int p = j < 27 ? j / 9 : j < 36 ? 3 + (j - 27) / 3 : j < 54 ? 9 + (j - 36) : -1;
      const int slot = j < 27 ? j % 9 : j < 36 ? (j - 27) % 3 : 0;
      if (ee >= nl || p < 0) CE[i] = 0.0;
      else if (async) cp_async8(CE + i, Et + (ee * P + p) * 9 + slot);
      else CE[i] = Et[(ee * P + p) * 9 + slot];
    }
  };
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t e0 = prm.e0 + tile * TE;
    const int64_t left = prm.e0 + prm.n - e0;
    const int ne = static_cast<int>(left < TE ? left : TE);
    const int el = x.e < ne ? x.e : ne - 1;
    x.ap = prm.aplus + (e0 + el) * 4 * P * 9;
    if (tid == 0 && tile + gridDim.x < ntiles) {  // next tile's streams -> L2 while this one computes
      const int64_t n0 = prm.e0 + (tile + gridDim.x) * TE;
      const int64_t nl = prm.e0 + prm.n - n0 < TE ? prm.e0 + prm.n - n0 : TE;
      l2_prefetch(prm.Q + n0 * P * B, nl * P * B * 8);
      l2_prefetch(prm.star + n0 * 3 * P * 3, nl * 3 * P * 3 * 8);
      l2_prefetch(prm.src + n0 * P * 9, nl * P * 9 * 8);
      l2_prefetch(prm.aplus + n0 * 4 * P * 9, nl * 4 * P * 9 * 8);
    }
    cp_async_wait_all();
    __syncthreads();  // previous tile done with every buffer; this tile's Q^n in Z
    {
#pragma unroll 4
      for (int i = tid; i < TE * P * B; i += NTH) {
        const int ee = i / (P * B), r = i - ee * P * B, p = r / B, kk = r - p * B;
        D[kk * SD + p * TE + ee] = ee < ne ? Z[i] : 0.0;
      }
      if (tile == blockIdx.x) coeffs(tile, false);  // later tiles: staged during the previous tile
    }
    __syncthreads();
    double I[P];
    if (comb) {
#pragma unroll
      for (int p = 0; p < P; ++p) I[p] = prm.dt * D[cr * SD + p * TE + cel];
    }
#pragma unroll 1
    for (int d = 0; d < N; ++d) {
      {
        double acc[3][V::NCK][2];
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int mt = 0; mt < V::NCK; ++mt) acc[c][mt][0] = acc[c][mt][1] = 0.0;
        ck<N>(x, acc);
        int rck[V::NCK];
        rows_of(V::ck_rows, ar, rck);
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int mt = 0; mt < V::NCK; ++mt)
            if (rck[mt] >= 0)
              st2(Z + (c * B + rck[mt]) * ZS + w * TE + ae, acc[c][mt][0], acc[c][mt][1]);
      }
      __syncthreads();  // Z complete, every warp done reading D^d
      if (comb) {
        const double s1 = prm.scal[d], s2 = prm.scal[N + d];
        const bool last = d + 1 == N;
        double* dr = D + cr * SD + cel;
        combine<B, false>(Z + cr * ZS + cel, dr, CS + cel * CSE, CE + cel * CEE, prm.wratio, [&](int p, double v) {
          v *= s1;
          I[p] = fma(s2, v, I[p]);
          dr[p * TE] = last ? I[p] : v;  // D^{d+1}; after the last step the time integral
        });
      }
      __syncthreads();
    }
    // volume (left-first) and the traces of the elastic columns, both from I
    double ta[4][V::NT][2];
    {
      double acc[3][V::NQ][2];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int mt = 0; mt < V::NQ; ++mt) acc[c][mt][0] = acc[c][mt][1] = 0.0;
      vol<N>(x, acc);
      int rq[V::NQ];
      rows_of(V::q_rows, ar, rq);
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int mt = 0; mt < V::NQ; ++mt)
          if (rq[mt] >= 0)
            st2(Z + (c * B + rq[mt]) * ZS + w * TE + ae, acc[c][mt][0], acc[c][mt][1]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int mt = 0; mt < V::NT; ++mt) ta[i][mt][0] = ta[i][mt][1] = 0.0;
    traces<N>(x, ta);
    __syncthreads();  // volume products complete
    if (comb) {  // volume result V[r][p][e] into the thread's own Z slots (c, t) = (p / 9, p % 9)
      double* zr = Z + cr * ZS + cel;
      combine<B, true>(zr, D + cr * SD + cel, CS + cel * CSE, CE + cel * CEE, prm.wratio,
                       [&](int p, double v) { zr[(p / 9) * B * ZS + (p % 9) * TE] = v; });
    }
    __syncthreads();  // I no longer read: the traces take the D buffer; CS / CE free
    if (tile + gridDim.x < ntiles) coeffs(tile + gridDim.x, true);
    {
      int rtr[V::NT];
      rows_of(V::tr_rows, ar, rtr);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int mt = 0; mt < V::NT; ++mt)
          if (rtr[mt] >= 0)
            *reinterpret_cast<double2*>(TR + (i * V::BtR + rtr[mt]) * TS + w * TE + ae) =
                make_double2(ta[i][mt][0], ta[i][mt][1]);
      for (int i = tid; i < 4 * (V::BtR - Bt) * 9 * TE; i += NTH) {  // padding rows of the traces
        const int f = i / ((V::BtR - Bt) * 9 * TE), r = i - f * (V::BtR - Bt) * 9 * TE;
        TR[(f * V::BtR + Bt + r / (9 * TE)) * TS + r % (9 * TE)] = 0.0;
      }
    }
    __syncthreads();
    {
      double* gt = prm.traces + e0 * 4 * Bt * 9;
      for (int i = tid; i < ne * 4 * Bt * 9; i += NTH) {
        const int ee = i / (4 * Bt * 9), r = i - ee * 4 * Bt * 9, f = r / (Bt * 9), mq = r - f * Bt * 9;
        const int m = mq / 9, qq = mq - m * 9;
        gt[i] = TR[(f * V::BtR + m) * TS + qq * TE + ee];
      }
    }
    // local flux lifted onto the volume result
    double qa[V::NQ][3][2];
    int rq[V::NQ];
    rows_of(V::q_rows, ar, rq);
#pragma unroll
    for (int mt = 0; mt < V::NQ; ++mt)
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        const int p = p0 + u;
        if (rq[mt] >= 0) {
          const double* v = Z + ((p / 9) * B + rq[mt]) * ZS + (p % 9) * TE + ae;
          qa[mt][u][0] = v[0];
          qa[mt][u][1] = v[TE * 0 + 1];
        } else {
          qa[mt][u][0] = qa[mt][u][1] = 0.0;
        }
      }
    lift<N>(x, qa);
    __syncthreads();  // every warp done reading the traces and Z
    if (tile + gridDim.x < ntiles) issue_q(tile + gridDim.x);
#pragma unroll
    for (int mt = 0; mt < V::NQ; ++mt)
#pragma unroll
      for (int u = 0; u < 3; ++u)
        if (rq[mt] >= 0)
          st2(D + rq[mt] * SD + (p0 + u) * TE + ae, qa[mt][u][0], qa[mt][u][1]);
    __syncthreads();
    double* Qw = prm.Q + e0 * P * B;
#if YDG_VQB
    {  // YDG_VQB: every Q^n load of the thread in flight at once (one memory latency)
      constexpr int NQ = (TE * P * B + NTH - 1) / NTH;
      const int n = ne * P * B;
      double qv[NQ];
#pragma unroll
      for (int j = 0; j < NQ; ++j) {
        const int i = tid + j * NTH;
        qv[j] = i < n ? Qw[i] : 0.0;
      }
#pragma unroll
      for (int j = 0; j < NQ; ++j) {
        const int i = tid + j * NTH;
        if (i < n) {
          const int ee = i / (P * B), r = i - ee * P * B, p = r / B, kk = r - p * B;
          Qw[i] = qv[j] + D[kk * SD + p * TE + ee];
        }
      }
    }
#else
#pragma unroll 4
    for (int i = tid; i < ne * P * B; i += NTH) {
      const int ee = i / (P * B), r = i - ee * P * B, p = r / B, kk = r - p * B;
      Qw[i] += D[kk * SD + p * TE + ee];
    }
#endif
  }
}

// Neighbour flux: Q += sum_i R^i (f^{h_i} T^{nb_i}_{j_i}) A-_i^T.
// Software-pipelined over the CTA's tiles: while tile t is rotated and lifted, the
// neighbours' traces of tile t+1 (cp.async, double-buffered), its Q^n and the neighbour
// slots of tile t+2 are in flight.  The rotation by f^h runs over dense degree-block
// windows; the lift (Y chunks + DMMA, as in the local kernel with A-) accumulates onto
// Q^n, and the result leaves through a shared staging block with coalesced stores.
template <int N>
constexpr int zsz() { return 4 * VT<N>::BtR * TS; }
template <int N>
constexpr int gsz() { return 4 * TE * VT<N>::Bt * 9; }
template <int N>
constexpr int fnz() { return 3 * VT<N>::Bt * VT<N>::Bt; }  // dense f^0..2
template <int N>
constexpr int nreg() {  // GT0 | Z | GT1 (the Q staging spans GT0+Z or Z+GT1) | QB
  return gsz<N>() + zsz<N>() + gsz<N>() + TE * P * VT<N>::B;
}
template <int N>
constexpr size_t nsmem_bytes() {
  static_assert(gsz<N>() + zsz<N>() >= TE * P * VT<N>::B, "Q staging fits GT + Z");
  return (static_cast<size_t>(VT<N>::NLIFTF) * 32 + nreg<N>() + 3 * 4 * TE + fnz<N>()) * sizeof(double) +
         (3 * 4 * TE + 3 * VT<N>::Bt + 1) * sizeof(int);
}


template <int N>
__global__ void __launch_bounds__(NTH, 1) vm_neigh(const GenParams prm) {
  using V = VT<N>;
  constexpr int B = V::B, Bt = V::Bt, BtR = V::BtR;
  extern __shared__ __align__(16) double sm[];
  double* FR = sm;                          // the lift's A fragments (table slots 0..NLIFTF-1)
  double* GT0 = FR + V::NLIFTF * 32;        // gathered neighbour traces [e][face][n][9], even tiles
  double* Z = GT0 + gsz<N>();               // rotated neighbour traces [4][BtR][TS]
  double* GT1 = Z + zsz<N>();               // odd tiles
  double* QB = GT1 + gsz<N>();              // the tile's Q^n, element-major as in HBM
  int64_t* NB = reinterpret_cast<int64_t*>(QB + TE * P * B);  // [3][e*4+face] neighbour ids
  double* FD = reinterpret_cast<double*>(NB + 3 * 4 * TE);      // f^h dense [h][m][n]
  int* JH = reinterpret_cast<int*>(FD + fnz<N>());             // [3][e*4+face] j | h << 2
  int* LO = JH + 3 * 4 * TE;                                   // per (h, m): first nonzero column
  int* WIDE = LO + 3 * Bt;                                     // any row wider than N + 1 columns
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = group_of(w), p0 = 3 * g;
  {
    const double* f = vfrag<N>();
    for (int i = tid; i < V::NLIFTF * 32; i += NTH) FR[i] = f[i];
    // f^h is block diagonal by degree (width <= N + 1 per row): dense rows + column windows
    if (tid == 0) *WIDE = 0;
    for (int i = tid; i < fnz<N>(); i += NTH) FD[i] = 0.0;
    __syncthreads();
    for (int row = tid; row < 3 * Bt; row += NTH) {
      int lo = Bt, hi = -1;
      for (int t = prm.f_ptr[row]; t < prm.f_ptr[row + 1]; ++t) {
        const int c = prm.f_col[t];
        FD[row * Bt + c] = prm.f_val[t];
        lo = c < lo ? c : lo;
        hi = c > hi ? c : hi;
      }
      if (hi < lo) lo = hi = 0;
      if (lo + N + 1 > Bt) lo = Bt - (N + 1) > 0 ? Bt - (N + 1) : 0;  // keep the window inside the row
      if (hi >= lo + N + 1) atomicOr(WIDE, 1);
      LO[row] = lo;
    }
  }
  Ctx<N> x;
  x.TR = Z;
  x.FR = FR;
  x.lane = lane;
  x.k = lane & 3;
  x.e = lane >> 2;
  x.p0 = p0;
  const int ar = lane >> 2, ae = 2 * (lane & 3);
  const int64_t ntiles = (prm.n + TE - 1) / TE;
  auto count = [&](int64_t t) {
    const int64_t n0 = prm.e0 + t * TE;
    return static_cast<int>(prm.e0 + prm.n - n0 < TE ? prm.e0 + prm.n - n0 : TE);
  };
  auto slots = [&](int64_t t, int buf) {  // neighbour ids / j|h of tile t -> slot buffer buf
    const int64_t n0 = prm.e0 + t * TE;
    if (tid < count(t) * 4) {
      cp_async8(NB + buf * 4 * TE + tid, prm.nb + n0 * 4 + tid);
      JH[buf * 4 * TE + tid] = prm.jh[n0 * 4 + tid];
    }
  };
  auto gathers = [&](int64_t t, int sbuf, double* gt) {
    const int64_t* nb = NB + sbuf * 4 * TE;
    const int* jh = JH + sbuf * 4 * TE;
    for (int i = tid; i < count(t) * 4 * Bt * 9; i += NTH) {
      const int ef = i / (Bt * 9), nq = i - ef * Bt * 9;
      cp_async8(gt + i, prm.traces + (nb[ef] * 4 + (jh[ef] & 3)) * Bt * 9 + nq);
    }
  };
  auto qload = [&](int64_t t) {
    const double* Qt = prm.Q + (prm.e0 + t * TE) * P * B;
    for (int i = tid; i < count(t) * P * B; i += NTH) cp_async8(QB + i, Qt + i);
  };
  if (blockIdx.x < ntiles) {  // prologue: slots of the first two tiles, traces + Q^n of the first
    slots(blockIdx.x, 0);
    cp_async_wait_all();
    __syncthreads();
    gathers(blockIdx.x, 0, GT0);
    qload(blockIdx.x);
    if (blockIdx.x + gridDim.x < ntiles) slots(blockIdx.x + gridDim.x, 1);
  }
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int cur = it & 1, sb = it % 3;
    double* GT = cur ? GT1 : GT0;
    double* QS = cur ? Z : GT0;  // Q staging: GT0 + Z or Z + GT1, never the next tile's GT
    const int64_t e0 = prm.e0 + tile * TE;
    const int ne = count(tile);
    const int el = x.e < ne ? x.e : ne - 1;
    x.ap = prm.aminus + (e0 + el) * 4 * P * 9;
    cp_async_wait_all();
    __syncthreads();  // traces + Q^n of this tile and the next tile's slots landed; staging free
    const int64_t nxt = tile + gridDim.x;
    if (nxt < ntiles) {
      gathers(nxt, (it + 1) % 3, cur ? GT0 : GT1);
      if (nxt + gridDim.x < ntiles) slots(nxt + gridDim.x, (it + 2) % 3);
      if (tid == 0) {
        const int64_t n0 = prm.e0 + nxt * TE;
        l2_prefetch(prm.Q + n0 * P * B, count(nxt) * P * B * 8);
        l2_prefetch(prm.aminus + n0 * 4 * P * 9, count(nxt) * 4 * P * 9 * 8);
      }
    }
    {
      const int* jh = JH + sb * 4 * TE;
      for (int i = tid; i < 4 * BtR * 9 * TE; i += NTH) {
        const int ee = i & (TE - 1), q = (i >> 3) % 9, fm = i / (9 * TE), m = fm % BtR, f = fm / BtR;
        double s = 0.0;
        if (m < Bt && ee < ne) {
          const int row = (jh[ee * 4 + f] >> 2) * Bt + m;
          const double* gt = GT + (ee * 4 + f) * Bt * 9 + q;
          const double* fr = FD + row * Bt;
          if (!*WIDE) {
            const int lo = LO[row];
#pragma unroll
            for (int n = 0; n <= N && n < Bt; ++n) s = fma(fr[lo + n], gt[(lo + n) * 9], s);
          } else {
            for (int n = 0; n < Bt; ++n) s = fma(fr[n], gt[n * 9], s);
          }
        }
        Z[(f * BtR + m) * TS + q * TE + ee] = s;
      }
    }
    // the lift accumulates onto Q^n (element-major in QB)
    double qa[V::NQ][3][2];
    int rq[V::NQ];
    rows_of(V::q_rows, ar, rq);
#pragma unroll
    for (int mt = 0; mt < V::NQ; ++mt)
#pragma unroll
      for (int u = 0; u < 3; ++u)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          qa[mt][u][h] = (rq[mt] >= 0 && ae + h < ne) ? QB[((ae + h) * P + p0 + u) * B + rq[mt]] : 0.0;
    __syncthreads();  // Z complete; QB read
    if (nxt < ntiles) qload(nxt);
    lift<N>(x, qa);
    __syncthreads();  // every warp done reading Z
#pragma unroll
    for (int mt = 0; mt < V::NQ; ++mt)
#pragma unroll
      for (int u = 0; u < 3; ++u)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (rq[mt] >= 0) QS[((ae + h) * P + p0 + u) * B + rq[mt]] = qa[mt][u][h];
    __syncthreads();
    double* Qw = prm.Q + e0 * P * B;
#pragma unroll 4
    for (int i = tid; i < ne * P * B; i += NTH) Qw[i] = QS[i];
  }
}

}  // namespace visco

bool visco_supported(int N, int P) { return P == 27 && N >= 1 && N <= 4; }

cudaError_t visco_configure(int N, const int (*scols)[3]) {
  // the kernel hard-codes the star column pattern; check it against the uploaded layout
  static const int vel[3][3] = {{0, 3, 5}, {3, 1, 4}, {5, 4, 2}};
  for (int p = 0; p < 27; ++p)
    for (int t = 0; t < 3; ++t)
      if (scols[p][t] != (p >= 6 && p < 9 ? vel[p - 6][t] : 6 + t)) return cudaErrorInvalidValue;
  cudaError_t e = cudaSuccess;
  switch (N) {
    case 1: e = cudaFuncSetAttribute(visco::vm_neigh<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(visco::nsmem_bytes<1>())); break;
    case 2: e = cudaFuncSetAttribute(visco::vm_neigh<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(visco::nsmem_bytes<2>())); break;
    case 3: e = cudaFuncSetAttribute(visco::vm_neigh<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(visco::nsmem_bytes<3>())); break;
    case 4: e = cudaFuncSetAttribute(visco::vm_neigh<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(visco::nsmem_bytes<4>())); break;
  }
  if (e != cudaSuccess) return e;
  switch (N) {
    case 1: return cudaFuncSetAttribute(visco::vm_local<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(visco::smem_bytes<1>()));
    case 2: return cudaFuncSetAttribute(visco::vm_local<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(visco::smem_bytes<2>()));
    case 3: return cudaFuncSetAttribute(visco::vm_local<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(visco::smem_bytes<3>()));
    case 4: return cudaFuncSetAttribute(visco::vm_local<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(visco::smem_bytes<4>()));
  }
  return cudaErrorInvalidValue;
}

cudaError_t visco_launch_neigh(const GenParams& p, cudaStream_t s) {
  const int64_t tiles = (p.n + visco::TE - 1) / visco::TE;
  if (tiles <= 0) return cudaSuccess;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const unsigned g = static_cast<unsigned>(tiles < sms ? tiles : sms);
  switch (p.N) {
    case 1: visco::vm_neigh<1><<<g, visco::NTH, visco::nsmem_bytes<1>(), s>>>(p); break;
    case 2: visco::vm_neigh<2><<<g, visco::NTH, visco::nsmem_bytes<2>(), s>>>(p); break;
    case 3: visco::vm_neigh<3><<<g, visco::NTH, visco::nsmem_bytes<3>(), s>>>(p); break;
    case 4: visco::vm_neigh<4><<<g, visco::NTH, visco::nsmem_bytes<4>(), s>>>(p); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t visco_launch_local(const GenParams& p, cudaStream_t s) {
  const int64_t tiles = (p.n + visco::TE - 1) / visco::TE;
  if (tiles <= 0) return cudaSuccess;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const unsigned g = static_cast<unsigned>(tiles < sms ? tiles : sms);
  switch (p.N) {
    case 1: visco::vm_local<1><<<g, visco::NTH, visco::smem_bytes<1>(), s>>>(p); break;
    case 2: visco::vm_local<2><<<g, visco::NTH, visco::smem_bytes<2>(), s>>>(p); break;
    case 3: visco::vm_local<3><<<g, visco::NTH, visco::smem_bytes<3>(), s>>>(p); break;
    case 4: visco::vm_local<4><<<g, visco::NTH, visco::smem_bytes<4>(), s>>>(p); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace ydg
