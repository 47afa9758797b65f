// LinA workload: ADER-DG-SEM for linearised acoustics on a uniform periodic cuboid grid
// (arXiv:1903.11521 §"LinA"; include/ydg_lina.h).  fp64, N + 1 <= 8 nodes per
// axis (Gauss-Lobatto), 4 quantities (p, u, v, w).
//
// Kernels (one element per CTA of 128 threads, persistent over elements; 4 CTAs per SM):
//   lina_local<N>  ADER predictor with the time integral accumulated in shared
//                  memory, volume term added to Q, side traces of I
//                  (X, Y, Z of P:1517-1521) written to HBM.
//   lina_flux<N>   local + neighbour flux of the six sides on the face nodes.
// A derivative along one axis is a dense (N+1) x (N+1) matrix applied to "pencils" of N+1
// nodes: a thread keeps a pencil in registers and does (N+1)^2 FMAs per N+1 shared loads,
// with the matrix entries as constant-bank operands.  The star matrices of acoustics have two
// nonzeros per axis (p <- u_a, u_a <- p), so a derivative needs six directional derivative
// fields (d_a p, d_a u_a), each written straight into its output quantity.
// Shared layout: quantity-major, node (x, y, z) at x*XS + y*YS + z with YS = N+2,
// XS = (N+1) YS (conflict-free y- and z-pencils at N+1 = 8).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ydg.h"
#include "../../include/ydg_lina.h"

namespace ydg {
namespace lina {

constexpr int kMaxN = 7;
constexpr int kT = 128;  // threads per CTA
#ifndef LINA_MINB
#define LINA_MINB 2  // CTAs per SM of lina_local: 2 with the register-resident I (12.6 ms) beat 3 (17.9, spills)
#endif

// Kt = -Dm (reading L4), Kh = W^-1 Dm^T W (L5), per order N (row-major n x n)
__constant__ double c_kt[kMaxN + 1][64];
__constant__ double c_kh[kMaxN + 1][64];
__constant__ double c_fh[kMaxN + 1][2];  // Fh^left_0, Fh^right_N (L6)

struct Params {
  double* Q;             // [e][p][x][y][z]
  double* traces;        // [e][6][p][u][v]  sides of I (u, v = the two other axes, ascending)
  const double* astar;   // [e][3][2] = (A*_a[0][1+a], A*_a[1+a][0])
  const double* aflux;   // [e][6][2][4][4] = A+ then A- per side (1/h folded in)
  const int32_t* nb;     // [e][6]
  int64_t ne;
  double dt;
  double tfac[kMaxN];    // dt^(d+2)/(d+2)!, d < N
};

template <int N>
struct Lay {
  static constexpr int n = N + 1, NN = n * n * n;
  // padded node space: YS odd and XS = 8 (mod 16) make the z- and y-pencil loads of a
  // half-warp hit 16 distinct double banks at n = 8
  static constexpr int YS = n + 1, XS = n * YS, NNP = n * XS;
  static constexpr int BUF = 4 * NNP;                               // one 4-quantity tensor
  static constexpr int SMEM = 3 * BUF + 4 * NN;                     // D, Dn, I, next Q (doubles)
  __device__ static int node(int x, int y, int z) { return x * XS + y * YS + z; }
};

// Out_{target} (=|+=) coef * sum_l M[k][l] S_{src}(pencil along axis a), for the pencil
// task t in [0, n^2): (u, v) = the other two axes.  ACC: add instead of store.
template <int N, int MAT>
__device__ __forceinline__ double mat(int k, int l) {
  // constant-cache load at the use (volatile: fewer matrix entries are kept live across the
  // element loop than with plain __constant__ reads: 76 vs 328 bytes of spills at N = 7)
  const double* p = (MAT == 0 ? c_kt[N] : c_kh[N]) + k * (N + 1) + l;
  unsigned long long a;
  asm("cvta.to.const.u64 %0, %1;" : "=l"(a) : "l"(p));
  double v;
  asm volatile("ld.const.f64 %0, [%1];" : "=d"(v) : "l"(a));
  return v;
}
template <int N, int AXIS, bool ACC, int MAT, bool IR>
__device__ __forceinline__ void pencil(const double* __restrict__ S, double* __restrict__ Out, int t, double coef,
                                       double (&ir)[N + 1], double f) {
  using L = Lay<N>;
  constexpr int n = L::n;
  const int u = t / n, v = t % n;
  int base, stride;
  if (AXIS == 0) { base = u * L::YS + v; stride = L::XS; }
  else if (AXIS == 1) { base = u * L::XS + v; stride = L::YS; }
  else { base = u * L::XS + v * L::YS; stride = 1; }
  double in[n], acc[n];
#pragma unroll
  for (int l = 0; l < n; ++l) in[l] = S[base + l * stride];
  // n independent accumulator chains (l outer): no dependent-FMA waits
#pragma unroll
  for (int k = 0; k < n; ++k) acc[k] = mat<N, MAT>(k, 0) * in[0];
#pragma unroll
  for (int l = 1; l < n; ++l)
#pragma unroll
    for (int k = 0; k < n; ++k) acc[k] = fma(mat<N, MAT>(k, l), in[l], acc[k]);
  double old[n];
  if (ACC)
#pragma unroll
    for (int k = 0; k < n; ++k) old[k] = Out[base + k * stride];
#pragma unroll
  for (int k = 0; k < n; ++k) {
    const double r = ACC ? fma(coef, acc[k], old[k]) : coef * acc[k];
    Out[base + k * stride] = r;
    if (IR) ir[k] = fma(f, r, ir[k]);  // the value is final: I += f D (registers)
  }
}

// node offset of pencil task t of `axis` at position k along it (the pencil() addressing)
template <int N, int AXIS>
__device__ __forceinline__ int pencil_node(int t, int k) {
  using L = Lay<N>;
  const int u = t / L::n, v = t % L::n;
  if (AXIS == 0) return u * L::YS + v + k * L::XS;
  if (AXIS == 1) return u * L::XS + v + k * L::YS;
  return u * L::XS + v * L::YS + k;
}

// Out = sum_a A*_a-mixing of (M along axis a) applied to S (P:1491-1496 / P:1506-1509):
//   Out_p = sum_a A*_a[0][1+a] (M_a S_{u_a}),   Out_{u_a} = A*_a[1+a][0] (M_a S_p).
// Three phases (one per axis); 2 n^2 pencil tasks per phase; barriers between phases
// (Out_p is accumulated).
template <int N, int MAT, bool IR>
__device__ __forceinline__ void apply3(const double* S, double* Out, const double (&c)[3][2], int tid,
                                       double (&ir)[3][N + 1], double f) {
  using L = Lay<N>;
  constexpr int n2 = L::n * L::n;
  const double* Sp = S;
  double* Op = Out;
  // IR: the time integral of every value once it is final lives in the registers of the
  // thread that finalises it (fixed task per thread: 2 n^2 <= 128 = kT): threads < n^2 hold
  // I_u (x phase), I_v (y), I_w (z) pencils, threads >= n^2 the I_p pencil (z phase)
  for (int t = tid; t < 2 * n2; t += kT) {  // axis x: d_x p -> u, d_x u -> p (store)
    if (t < n2) pencil<N, 0, false, MAT, IR>(Sp, Out + 1 * L::NNP, t, c[0][1], ir[0], f);
    else pencil<N, 0, false, MAT, false>(S + 1 * L::NNP, Op, t - n2, c[0][0], ir[0], f);
  }
  __syncthreads();
  for (int t = tid; t < 2 * n2; t += kT) {  // axis y: d_y p -> v, d_y v -> p (+=)
    if (t < n2) pencil<N, 1, false, MAT, IR>(Sp, Out + 2 * L::NNP, t, c[1][1], ir[1], f);
    else pencil<N, 1, true, MAT, false>(S + 2 * L::NNP, Op, t - n2, c[1][0], ir[0], f);
  }
  __syncthreads();
  for (int t = tid; t < 2 * n2; t += kT) {  // axis z: d_z p -> w, d_z w -> p (+=)
    if (t < n2) pencil<N, 2, false, MAT, IR>(Sp, Out + 3 * L::NNP, t, c[2][1], ir[2], f);
    else pencil<N, 2, true, MAT, IR>(S + 3 * L::NNP, Op, t - n2, c[2][0], ir[0], f);
  }
  __syncthreads();
}

// The thread's register pencils of I <-> the shared I tensor (see apply3).
template <int N, bool TO_SHARED>
__device__ __forceinline__ void ireg_io(double* I, double (&ir)[3][N + 1], int tid, double scale) {
  using L = Lay<N>;
  constexpr int n = L::n, n2 = n * n;
  if (tid < n2) {
#pragma unroll
    for (int k = 0; k < n; ++k) {
      const int a = 1 * L::NNP + pencil_node<N, 0>(tid, k), b = 2 * L::NNP + pencil_node<N, 1>(tid, k),
                c = 3 * L::NNP + pencil_node<N, 2>(tid, k);
      if (TO_SHARED) { I[a] = ir[0][k]; I[b] = ir[1][k]; I[c] = ir[2][k]; }
      else { ir[0][k] = scale * I[a]; ir[1][k] = scale * I[b]; ir[2][k] = scale * I[c]; }
    }
  } else if (tid < 2 * n2) {
#pragma unroll
    for (int k = 0; k < n; ++k) {
      const int a = pencil_node<N, 2>(tid - n2, k);
      if (TO_SHARED) I[a] = ir[0][k];
      else ir[0][k] = scale * I[a];
    }
  }
}

template <int N>
__global__ void __launch_bounds__(kT, LINA_MINB) lina_local(const __grid_constant__ Params prm) {
  using L = Lay<N>;
  constexpr int n = L::n, NN = L::NN;
  extern __shared__ __align__(16) double sm[];
  double* D = sm;
  double* Dn = sm + L::BUF;
  double* I = sm + 2 * L::BUF;
  double* R = sm + 3 * L::BUF;  // Q of the next element, canonical order (cp.async prefetch)
  const int tid = threadIdx.x;
  auto prefetch = [&](int64_t e) {  // 16-byte cp.async chunks of element e's Q into R
    const double* src = prm.Q + e * 4 * NN;
    for (int c = tid; c < 2 * NN; c += kT)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(R + 2 * c))),
                   "l"(src + 2 * c)
                   : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (blockIdx.x < prm.ne) prefetch(blockIdx.x);
  for (int64_t e = blockIdx.x; e < prm.ne; e += gridDim.x) {
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();  // R holds Q of element e
#pragma unroll 4
    for (int i = tid; i < 4 * NN; i += kT) {
      const int q = i / NN, r = i % NN, x = r / (n * n), y = (r / n) % n, z = r % n;
      D[q * L::NNP + L::node(x, y, z)] = R[i];
    }
    __syncthreads();  // R is free: the next element's Q streams in during this one
    if (e + gridDim.x < prm.ne) prefetch(e + gridDim.x);
    double c[3][2];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      c[a][0] = prm.astar[(e * 3 + a) * 2];
      c[a][1] = prm.astar[(e * 3 + a) * 2 + 1];
    }
    __syncthreads();
    double ir[3][n];
    ireg_io<N, false>(D, ir, tid, prm.dt);  // I = dt D^0, in registers
    double* cur = D;
    double* nxt = Dn;
    for (int d = 0; d < N; ++d) {  // CK recursion and time integral
      apply3<N, 0, true>(cur, nxt, c, tid, ir, prm.tfac[d]);
      double* t = cur;
      cur = nxt;
      nxt = t;
    }
    ireg_io<N, true>(I, ir, tid, 1.0);
    __syncthreads();
    apply3<N, 1, false>(I, nxt, c, tid, ir, 0.0);  // volume into nxt
    // Q* = Q + volume; sides of I -> traces
    double* Qw = prm.Q + e * 4 * NN;
    constexpr int QIT = (4 * NN + kT - 1) / kT;
    {  // Q* = Q + volume: all of the thread's Q loads in flight at once
      double qv[QIT];
#pragma unroll
      for (int j = 0; j < QIT; ++j) {
        const int i = tid + j * kT;
        qv[j] = i < 4 * NN ? Qw[i] : 0.0;
      }
#pragma unroll
      for (int j = 0; j < QIT; ++j) {
        const int i = tid + j * kT;
        if (i < 4 * NN) {
          const int q = i / NN, r = i % NN, s = q * L::NNP + L::node(r / (n * n), (r / n) % n, r % n);
          Qw[i] = qv[j] + nxt[s];
        }
      }
    }
    double* Te = prm.traces + e * 6 * 4 * n * n;
    for (int i = tid; i < 6 * 4 * n * n; i += kT) {
      const int side = i / (4 * n * n), r = i % (4 * n * n), q = r / (n * n), u = (r / n) % n, v = r % n;
      const int a = side >> 1, at = (side & 1) ? N : 0;
      const int node = a == 0 ? L::node(at, u, v) : (a == 1 ? L::node(u, at, v) : L::node(u, v, at));
      Te[i] = I[q * L::NNP + node];
    }
    __syncthreads();  // before the next element overwrites the shared tensors
  }
}

// Local + neighbour flux of the six sides on the face nodes of each element:
// F = (A+)^s X^s + (A-)^s X^Neigh(s) (4 x 4 each), Q[face node] += Fh^s F.  Three phases
// (x, y, z sides) so that edge and corner nodes are updated by one thread at a time.
template <int N>
__global__ void __launch_bounds__(kT) lina_flux(const __grid_constant__ Params prm) {
  constexpr int n = N + 1, NN = n * n * n, n2 = n * n;
  const int tid = threadIdx.x;
  const double fl = c_fh[N][0], fr = c_fh[N][1];
  for (int64_t e = blockIdx.x; e < prm.ne; e += gridDim.x) {
    double* Qe = prm.Q + e * 4 * NN;
    const double* Te = prm.traces + e * 6 * 4 * n2;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      for (int t = tid; t < 2 * n2; t += kT) {
        const int end = t / n2, r = t % n2, u = r / n, v = r % n, side = 2 * a + end;
        const int opp = side ^ 1;
        const int64_t nbe = prm.nb[e * 6 + side];
        const double* To = Te + side * 4 * n2 + r;
        const double* Tn = prm.traces + (nbe * 6 + opp) * 4 * n2 + r;
        double xo[4], xn[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          xo[q] = To[q * n2];
          xn[q] = Tn[q * n2];
        }
        const double* Ap = prm.aflux + ((e * 6 + side) * 2) * 16;
        const double* Am = Ap + 16;
        const int at = end ? N : 0;
        const int node = a == 0 ? (at * n + u) * n + v : (a == 1 ? (u * n + at) * n + v : (u * n + v) * n + at);
        const double fh = end ? fr : fl;
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          double s = 0.0;
#pragma unroll
          for (int q = 0; q < 4; ++q) s = fma(Ap[p * 4 + q], xo[q], fma(Am[p * 4 + q], xn[q], s));
          Qe[p * NN + node] = fma(fh, s, Qe[p * NN + node]);
        }
      }
      __syncthreads();  // edge / corner nodes of the next axis
    }
  }
}

}  // namespace lina
}  // namespace ydg

// ------------------------------------------------------------------ host side (C ABI)

struct ydg_lina {
  int N = 0, dev = 0;
  int status = 0;
  std::string err;
  cudaStream_t stream = nullptr;
  int nx = 0, ny = 0, nz = 0;
  int64_t ne = 0;
  double* Q = nullptr;
  double* traces = nullptr;
  double* astar = nullptr;
  double* aflux = nullptr;
  int32_t* nb = nullptr;
  size_t bytes = 0;
  int grid = 0, grid_flux = 0;
};

namespace {

using ydg::lina::kMaxN;

int lfail(ydg_lina* h, int code, const std::string& msg) {
  h->err = msg;
  if (code == YDG_ERR_CUDA) h->status = code;
  return code;
}
#define LCUDA(h, call)                                                                  \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return lfail(h, e_ == cudaErrorMemoryAllocation ? YDG_ERR_OOM : YDG_ERR_CUDA,     \
                   std::string(#call) + ": " + cudaGetErrorString(e_));                 \
  } while (0)

// Gauss-Lobatto-Legendre nodes / weights on [0, 1] in long double (Newton on P_N' from
// Chebyshev-Lobatto starts; the library's own construction, independent of the oracle's)
void gll(int N, std::vector<long double>& x, std::vector<long double>& w) {
  x.assign(N + 1, 0.0L);
  w.assign(N + 1, 0.0L);
  auto legendre = [N](long double t, long double& P, long double& dP, long double& d2P) {
    long double p0 = 1.0L, p1 = t;
    if (N == 0) { P = 1; dP = 0; d2P = 0; return; }
    for (int k = 2; k <= N; ++k) {
      const long double p2 = ((2 * k - 1) * t * p1 - (k - 1) * p0) / k;
      p0 = p1;
      p1 = p2;
    }
    P = p1;
    // (1 - t^2) P' = N (P_{N-1} - t P_N);  (1 - t^2) P'' = 2 t P' - N (N + 1) P
    dP = N * (p0 - t * p1) / (1.0L - t * t);
    d2P = (2.0L * t * dP - N * (N + 1.0L) * p1) / (1.0L - t * t);
  };
  const long double pi = 3.14159265358979323846264338327950288L;
  for (int i = 0; i <= N; ++i) {
    long double t = -std::cos(pi * i / N);
    if (i > 0 && i < N) {
      for (int it = 0; it < 100; ++it) {
        long double P, dP, d2P;
        legendre(t, P, dP, d2P);
        const long double dt = dP / d2P;
        t -= dt;
        if (std::fabs(dt) < 1e-30L) break;
      }
    }
    long double P, dP, d2P;
    legendre(t, P, dP, d2P);
    x[i] = (t + 1.0L) / 2.0L;
    w[i] = 1.0L / (N * (N + 1.0L) * P * P);  // 2 / (N (N+1) P^2) on [-1,1], halved
  }
}

}  // namespace

static void lina_free(ydg_lina* h) {
  for (void** p : {reinterpret_cast<void**>(&h->Q), reinterpret_cast<void**>(&h->traces),
                   reinterpret_cast<void**>(&h->astar), reinterpret_cast<void**>(&h->aflux),
                   reinterpret_cast<void**>(&h->nb)}) {
    if (*p) cudaFree(*p);
    *p = nullptr;
  }
  h->bytes = 0;
  h->ne = 0;
}

template <int N>
static size_t local_smem() { return sizeof(double) * ydg::lina::Lay<N>::SMEM; }
static size_t smem_of(int N) {
  switch (N) {
    case 1: return local_smem<1>();
    case 2: return local_smem<2>();
    case 3: return local_smem<3>();
    case 4: return local_smem<4>();
    case 5: return local_smem<5>();
    case 6: return local_smem<6>();
    default: return local_smem<7>();
  }
}
static const void* local_fn(int N) {
  switch (N) {
    case 1: return reinterpret_cast<const void*>(&ydg::lina::lina_local<1>);
    case 2: return reinterpret_cast<const void*>(&ydg::lina::lina_local<2>);
    case 3: return reinterpret_cast<const void*>(&ydg::lina::lina_local<3>);
    case 4: return reinterpret_cast<const void*>(&ydg::lina::lina_local<4>);
    case 5: return reinterpret_cast<const void*>(&ydg::lina::lina_local<5>);
    case 6: return reinterpret_cast<const void*>(&ydg::lina::lina_local<6>);
    default: return reinterpret_cast<const void*>(&ydg::lina::lina_local<7>);
  }
}
static const void* flux_fn(int N) {
  switch (N) {
    case 1: return reinterpret_cast<const void*>(&ydg::lina::lina_flux<1>);
    case 2: return reinterpret_cast<const void*>(&ydg::lina::lina_flux<2>);
    case 3: return reinterpret_cast<const void*>(&ydg::lina::lina_flux<3>);
    case 4: return reinterpret_cast<const void*>(&ydg::lina::lina_flux<4>);
    case 5: return reinterpret_cast<const void*>(&ydg::lina::lina_flux<5>);
    case 6: return reinterpret_cast<const void*>(&ydg::lina::lina_flux<6>);
    default: return reinterpret_cast<const void*>(&ydg::lina::lina_flux<7>);
  }
}

static int lina_xfer(ydg_lina* h, int64_t first, int64_t count, const double* src, double* dst) {
  if (!h) return YDG_ERR_ARG;
  if (h->status) return h->status;
  if (!h->ne) return lfail(h, YDG_ERR_STATE, "upload the grid first");
  if (first < 0 || count < 0 || first + count > h->ne || (!src && !dst)) return lfail(h, YDG_ERR_ARG, "bad element range");
  const int n = h->N + 1;
  const size_t per = static_cast<size_t>(4) * n * n * n;
  LCUDA(h, cudaStreamSynchronize(h->stream));
  LCUDA(h, cudaDeviceSynchronize());
  if (src) LCUDA(h, cudaMemcpy(h->Q + first * per, src, count * per * sizeof(double), cudaMemcpyHostToDevice));
  else LCUDA(h, cudaMemcpy(dst, h->Q + first * per, count * per * sizeof(double), cudaMemcpyDeviceToHost));
  return YDG_OK;
}

extern "C" {

int ydg_lina_create(int order, int precision, int cuda_device, ydg_lina** out) {
  if (!out) return YDG_ERR_ARG;
  *out = nullptr;
  if (order < 1 || order > kMaxN) return YDG_ERR_UNSUPPORTED;
  if (precision != 8) return YDG_ERR_UNSUPPORTED;
  ydg_lina* h = new ydg_lina;
  h->N = order;
  h->dev = cuda_device;
  const int n = order + 1;
  std::vector<long double> x, w;
  gll(order, x, w);
  // Lagrange derivative matrix Dm_kl = psi'_l(x_k) (barycentric weights)
  std::vector<long double> lam(n, 1.0L);
  for (int j = 0; j < n; ++j)
    for (int m = 0; m < n; ++m)
      if (m != j) lam[j] /= (x[j] - x[m]);
  std::vector<long double> Dm(n * n, 0.0L);
  for (int k = 0; k < n; ++k) {
    long double diag = 0.0L;
    for (int l = 0; l < n; ++l)
      if (l != k) {
        Dm[k * n + l] = (lam[l] / lam[k]) / (x[k] - x[l]);
        diag -= Dm[k * n + l];
      }
    Dm[k * n + k] = diag;
  }
  double kt[64] = {0}, kh[64] = {0}, fh[2];
  for (int k = 0; k < n; ++k)
    for (int l = 0; l < n; ++l) {
      kt[k * n + l] = static_cast<double>(-Dm[k * n + l]);
      kh[k * n + l] = static_cast<double>(w[l] * Dm[l * n + k] / w[k]);
    }
  fh[0] = static_cast<double>(-1.0L / w[0]);
  fh[1] = static_cast<double>(-1.0L / w[order]);
  cudaError_t e = cudaSetDevice(cuda_device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(ydg::lina::c_kt, kt, sizeof(kt), sizeof(kt) * order);
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(ydg::lina::c_kh, kh, sizeof(kh), sizeof(kh) * order);
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(ydg::lina::c_fh, fh, sizeof(fh), sizeof(fh) * order);
  if (e != cudaSuccess) {
    delete h;
    return YDG_ERR_CUDA;
  }
  *out = h;
  return YDG_OK;
}

int ydg_lina_upload_grid(ydg_lina* h, int nx, int ny, int nz, const double* hxyz, const double* material) {
  if (!h) return YDG_ERR_ARG;
  if (h->status) return h->status;
  if (nx < 1 || ny < 1 || nz < 1 || !hxyz || !material) return lfail(h, YDG_ERR_ARG, "bad grid");
  if (!(hxyz[0] > 0 && hxyz[1] > 0 && hxyz[2] > 0)) return lfail(h, YDG_ERR_ARG, "cell sizes must be > 0");
  const int64_t E = static_cast<int64_t>(nx) * ny * nz;
  if (E > INT32_MAX) return lfail(h, YDG_ERR_UNSUPPORTED, "more than 2^31 elements");
  for (int64_t e = 0; e < E; ++e)
    if (!(material[2 * e] > 0 && material[2 * e + 1] > 0)) return lfail(h, YDG_ERR_ARG, "rho, K must be > 0");
  LCUDA(h, cudaSetDevice(h->dev));
  lina_free(h);
  const int n = h->N + 1;
  // neighbours (reading L8) and coefficients
  std::vector<int32_t> nb(E * 6);
  std::vector<double> astar(E * 6), aflux(E * 6 * 2 * 16, 0.0);
  for (int64_t e = 0; e < E; ++e) {
    const int64_t i = e % nx, j = (e / nx) % ny, k = e / (static_cast<int64_t>(nx) * ny);
    auto id = [&](int64_t a, int64_t b, int64_t c) {
      a = (a + nx) % nx;
      b = (b + ny) % ny;
      c = (c + nz) % nz;
      return static_cast<int32_t>(a + nx * (b + ny * c));
    };
    const int32_t nbs[6] = {id(i - 1, j, k), id(i + 1, j, k), id(i, j - 1, k), id(i, j + 1, k), id(i, j, k - 1), id(i, j, k + 1)};
    const double rho = material[2 * e], K = material[2 * e + 1];
    for (int a = 0; a < 3; ++a) {
      astar[(e * 3 + a) * 2] = K / hxyz[a];          // A*_a[0][1+a]
      astar[(e * 3 + a) * 2 + 1] = 1.0 / (rho * hxyz[a]);  // A*_a[1+a][0]
    }
    for (int s = 0; s < 6; ++s) {
      nb[e * 6 + s] = nbs[s];
      const int a = s >> 1;
      const double sg = (s & 1) ? 1.0 : -1.0;  // outward normal n = sg e_a
      const double rp = material[2 * nbs[s]], Kp = material[2 * nbs[s] + 1];
      const double Zm = std::sqrt(rho * K), Zp = std::sqrt(rp * Kp), S = Zm + Zp;
      // Godunov interface state (reading L7): p* = (Zp p- + Zm p+ + Zm Zp (un- - un+)) / S,
      // un* = (Zm un- + Zp un+ + p- - p+) / S; flux F = (K- un*, p* n / rho-), scaled 1/h_a
      double* Ap = &aflux[((e * 6 + s) * 2) * 16];
      double* Am = Ap + 16;
      const double ih = 1.0 / hxyz[a];
      // row p (0): K- un*
      Ap[0 * 4 + 0] = ih * K * (1.0 / S);
      Ap[0 * 4 + 1 + a] = ih * K * (Zm / S) * sg;
      Am[0 * 4 + 0] = ih * K * (-1.0 / S);
      Am[0 * 4 + 1 + a] = ih * K * (Zp / S) * sg;
      // row u_a (1 + a): sg p* / rho-
      Ap[(1 + a) * 4 + 0] = ih * sg / rho * (Zp / S);
      Ap[(1 + a) * 4 + 1 + a] = ih * sg / rho * (Zm * Zp / S) * sg;
      Am[(1 + a) * 4 + 0] = ih * sg / rho * (Zm / S);
      Am[(1 + a) * 4 + 1 + a] = ih * sg / rho * (-Zm * Zp / S) * sg;
    }
  }
  h->nx = nx;
  h->ny = ny;
  h->nz = nz;
  const size_t qb = static_cast<size_t>(E) * 4 * n * n * n * sizeof(double);
  const size_t tb = static_cast<size_t>(E) * 6 * 4 * n * n * sizeof(double);
  LCUDA(h, cudaMalloc(&h->Q, qb));
  LCUDA(h, cudaMalloc(&h->traces, tb));
  LCUDA(h, cudaMalloc(&h->astar, astar.size() * sizeof(double)));
  LCUDA(h, cudaMalloc(&h->aflux, aflux.size() * sizeof(double)));
  LCUDA(h, cudaMalloc(&h->nb, nb.size() * sizeof(int32_t)));
  h->bytes = qb + tb + (astar.size() + aflux.size()) * sizeof(double) + nb.size() * sizeof(int32_t);
  LCUDA(h, cudaMemset(h->Q, 0, qb));
  LCUDA(h, cudaMemset(h->traces, 0, tb));
  LCUDA(h, cudaMemcpy(h->astar, astar.data(), astar.size() * sizeof(double), cudaMemcpyHostToDevice));
  LCUDA(h, cudaMemcpy(h->aflux, aflux.data(), aflux.size() * sizeof(double), cudaMemcpyHostToDevice));
  LCUDA(h, cudaMemcpy(h->nb, nb.data(), nb.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  LCUDA(h, cudaFuncSetAttribute(local_fn(h->N), cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_of(h->N))));
  LCUDA(h, cudaFuncSetAttribute(local_fn(h->N), cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  int sms = 148, occ = 1, occf = 1;
  LCUDA(h, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->dev));
  LCUDA(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, local_fn(h->N), ydg::lina::kT, smem_of(h->N)));
  LCUDA(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occf, flux_fn(h->N), ydg::lina::kT, 0));
  h->grid = sms * std::max(1, occ);
  h->grid_flux = sms * std::max(1, occf);  // the flux kernel is latency-bound: every resident CTA
  h->ne = E;
  return YDG_OK;
}

int ydg_lina_upload_dofs(ydg_lina* h, int64_t first, int64_t count, const double* Q) {
  if (!Q) return h ? lfail(h, YDG_ERR_ARG, "null Q") : YDG_ERR_ARG;
  return lina_xfer(h, first, count, Q, nullptr);
}
int ydg_lina_download_dofs(ydg_lina* h, int64_t first, int64_t count, double* Q_out) {
  if (!Q_out) return h ? lfail(h, YDG_ERR_ARG, "null Q_out") : YDG_ERR_ARG;
  return lina_xfer(h, first, count, nullptr, Q_out);
}

int ydg_lina_step(ydg_lina* h, double dt, int nsteps, void* cuda_stream) {
  if (!h) return YDG_ERR_ARG;
  if (h->status) return h->status;
  if (!h->ne) return lfail(h, YDG_ERR_STATE, "upload the grid first");
  if (!(dt > 0) || !std::isfinite(dt) || nsteps < 0) return lfail(h, YDG_ERR_ARG, "bad dt or nsteps");
  cudaStream_t s = cuda_stream ? static_cast<cudaStream_t>(cuda_stream) : h->stream;
  ydg::lina::Params p{};
  p.Q = h->Q;
  p.traces = h->traces;
  p.astar = h->astar;
  p.aflux = h->aflux;
  p.nb = h->nb;
  p.ne = h->ne;
  p.dt = dt;
  double f = dt;
  for (int d = 0; d < h->N; ++d) {
    f *= dt / (d + 2);  // dt^(d+2) / (d+2)!
    p.tfac[d] = f;
  }
  void* args[] = {&p};
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(h->grid, h->ne));
  const unsigned gridf = static_cast<unsigned>(std::min<int64_t>(h->grid_flux, h->ne));
  for (int k = 0; k < nsteps; ++k) {
    LCUDA(h, cudaLaunchKernel(local_fn(h->N), dim3(grid), dim3(ydg::lina::kT), args, smem_of(h->N), s));
    LCUDA(h, cudaLaunchKernel(flux_fn(h->N), dim3(gridf), dim3(ydg::lina::kT), args, 0, s));
  }
  return YDG_OK;
}

int ydg_lina_query(ydg_lina* h, int what, double* v) {
  if (!h || !v) return YDG_ERR_ARG;
  const double n = h->N + 1, n3 = n * n * n, n2 = n * n;
  // nonzero flops per element-update (paper's rule; strength-reduced order):
  //   one derivative / volume term: per axis (D A*^T: 2 n^3 products) + (Kt on the two
  //   nonzero columns: 2 n^3 (2 n - 1)) + summing the 3 axes into p (2 n^3)
  //   time integral: 2 * 4 n^3 per derivative; Q update 4 n^3; flux: 6 sides x n^2 x
  //   (A+ and A- with 4 nonzeros each: 2 x (4 + 2) + 4 adds, Fh scaling 4 + update 4)
  const double deriv = 3 * (2 * n3 + 2 * n3 * (2 * n - 1)) + 2 * n3;
  const double flops = h->N * (deriv + 8 * n3) + deriv + 4 * n3 + 6 * n2 * (2 * 6 + 4 + 8);
  switch (what) {
    case 0: *v = static_cast<double>(h->ne); break;
    case 1: *v = flops; break;
    case 2: *v = 8.0 * (2 * 4 * n3 + 6 + 6 * 4 * n2 + 2 * 4 * n3 + 2 * 6 * 4 * n2 + 6 * 32) + 4.0 * 6; break;
    case 3: *v = static_cast<double>(h->bytes); break;
    case 4: *v = 2; break;
    default: return lfail(h, YDG_ERR_ARG, "unknown query");
  }
  return YDG_OK;
}

const char* ydg_lina_error_string(const ydg_lina* h) { return h ? h->err.c_str() : "null handle"; }

void ydg_lina_destroy(ydg_lina* h) {
  if (!h) return;
  cudaSetDevice(h->dev);
  if (h->stream) cudaStreamSynchronize(h->stream);
  lina_free(h);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

}  // extern "C"
