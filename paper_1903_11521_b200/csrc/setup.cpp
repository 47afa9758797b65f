// Host-side setup of the ADER-DG element update (fp64).  See setup.h.
//
// Geometry ("element-dependent linear combinations of the Jacobians"):
//   J = [x1-x0 | x2-x0 | x3-x0],  A*^c = sum_d (J^-1)_cd A^d.
// Flux solvers ("solution to the 1D Riemann problem", reading R8):
//   Godunov state of the face-normal elastic interface problem with both materials,
//   A+ = T Ax(m-) G- T^-1, A- = T Ax(m-) G+ T^-1, scaled by -2|S_i|/det J (reading R4).
// Viscoelastic extension (reading R14): memory variables theta^l rotate like stress and
// obey d_t theta^l - omega_l eps(v) = -omega_l theta^l; source E couples them back.
#include "setup.h"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>

namespace ydg {

namespace {

enum { SXX = 0, SYY, SZZ, SXY, SYZ, SXZ, VU, VV, VW };

// Voigt pairs (xx, yy, zz, xy, yz, xz)
constexpr int kVi[6] = {0, 1, 2, 0, 1, 0};
constexpr int kVj[6] = {0, 1, 2, 1, 2, 2};

int voigt(int i, int j) {
  if (i > j) std::swap(i, j);
  if (i == j) return i;
  if (i == 0 && j == 1) return 3;
  if (i == 1 && j == 2) return 4;
  return 5;
}

// Elastic Jacobian along axis d (0,1,2) for d_t q + sum_d A^d d_d q = 0, plus the
// memory-variable rows for P = 27 (omega per mechanism).
void jacobian(int P, int d, double rho, double lam, double mu, const double* omega, double* A) {
  std::fill(A, A + P * P, 0.0);
  auto at = [&](int r, int c) -> double& { return A[r * P + c]; };
  const double l2m = lam + 2.0 * mu, ir = 1.0 / rho;
  const int vel[3] = {VU, VV, VW};
  // normal stresses: d_t s_ii = lam div v + 2 mu d_i v_i
  for (int i = 0; i < 3; ++i) at(i, vel[d]) = -(i == d ? l2m : lam);
  // shear stresses: d_t s_ij = mu (d_i v_j + d_j v_i)
  for (int s = 3; s < 6; ++s) {
    const int i = kVi[s], j = kVj[s];
    if (d == i) at(s, vel[j]) = -mu;
    if (d == j) at(s, vel[i]) = -mu;
  }
  // velocities: rho d_t v_i = sum_m d_m s_im
  for (int i = 0; i < 3; ++i) at(vel[i], voigt(i, d)) = -ir;
  if (P == 27) {
    for (int l = 0; l < 3; ++l)
      for (int s = 0; s < 6; ++s) {
        const int i = kVi[s], j = kVj[s], row = 9 + 6 * l + s;
        // eps_ij = (d_i v_j + d_j v_i) / 2
        if (i == j) {
          if (d == i) at(row, vel[i]) = -omega[l];
        } else {
          if (d == i) at(row, vel[j]) += -0.5 * omega[l];
          if (d == j) at(row, vel[i]) += -0.5 * omega[l];
        }
      }
  }
}

void matmul(int P, const double* A, const double* B, double* C) {
  for (int i = 0; i < P; ++i)
    for (int j = 0; j < P; ++j) {
      double s = 0.0;
      for (int k = 0; k < P; ++k) s += A[i * P + k] * B[k * P + j];
      C[i * P + j] = s;
    }
}

// Quantity rotation for the frame R (columns n, s, t): q_global = T q_face.
void rotation(int P, const double R[3][3], double* T) {
  std::fill(T, T + P * P, 0.0);
  const int ntens = P == 27 ? 4 : 1;
  for (int b = 0; b < ntens; ++b) {
    const int base = b == 0 ? 0 : 9 + 6 * (b - 1);
    // S_g(ij) = sum_kl R_ik R_jl S_f(kl); a face-frame Voigt entry (k,l), k != l, stands
    // for both S_f(kl) and S_f(lk).
    for (int s = 0; s < 6; ++s)
      for (int f = 0; f < 6; ++f) {
        const int i = kVi[s], j = kVj[s], k = kVi[f], l = kVj[f];
        double v = R[i][k] * R[j][l];
        if (k != l) v += R[i][l] * R[j][k];
        T[(base + s) * P + base + f] = v;
      }
  }
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k) T[(6 + i) * P + 6 + k] = R[i][k];
}

void face_frame(const double n[3], double R[3][3]) {
  double a[3] = {1.0, 0.0, 0.0};
  if (std::fabs(n[0]) >= 0.9) { a[0] = 0.0; a[1] = 1.0; }
  const double dn = a[0] * n[0] + a[1] * n[1] + a[2] * n[2];
  double s[3] = {a[0] - dn * n[0], a[1] - dn * n[1], a[2] - dn * n[2]};
  const double ns = std::sqrt(s[0] * s[0] + s[1] * s[1] + s[2] * s[2]);
  for (double& x : s) x /= ns;
  const double t[3] = {n[1] * s[2] - n[2] * s[1], n[2] * s[0] - n[0] * s[2], n[0] * s[1] - n[1] * s[0]};
  for (int i = 0; i < 3; ++i) { R[i][0] = n[i]; R[i][1] = s[i]; R[i][2] = t[i]; }
}

struct Mat { double rho, lam, mu; };

Mat material_of(const double* m) {
  const double rho = m[0], vp = m[1], vs = m[2];
  const double mu = rho * vs * vs;
  return {rho, rho * vp * vp - 2.0 * mu, mu};
}

}  // namespace

void star_cols(int P, int p, int cols[3]) {
  static const int el[9][3] = {{VU, VV, VW}, {VU, VV, VW}, {VU, VV, VW},  {VU, VV, VV},
                               {VV, VW, VW}, {VU, VW, VW}, {SXX, SXY, SXZ}, {SXY, SYY, SYZ},
                               {SXZ, SYZ, SZZ}};
  const int r = p < 9 ? p : (p - 9) % 6;
  // viscoelastic: every non-velocity row on (VU, VV, VW) in order (zero where a shear row has
  // no entry), so the tensor-core kernel's star chunks read three fixed columns
  const bool vcols = P == 27 && (r < 6);
  for (int k = 0; k < 3; ++k) cols[k] = vcols ? VU + k : el[r][k];
}

bool match_faces(int64_t ne, const int64_t* vid, Neighbours* out, std::string* err) {
  struct Key { int64_t a, b, c; int64_t ef; };
  std::vector<Key> keys(static_cast<size_t>(ne) * 4);
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < ne; ++e)
    for (int i = 0; i < 4; ++i) {
      int64_t v[3] = {vid[e * 4 + kFaces[i][0]], vid[e * 4 + kFaces[i][1]], vid[e * 4 + kFaces[i][2]]};
      std::sort(v, v + 3);
      keys[e * 4 + i] = {v[0], v[1], v[2], e * 4 + i};
    }
  for (int64_t e = 0; e < ne; ++e)
    for (int a = 0; a < 4; ++a) {
      if (vid[e * 4 + a] < 0) { *err = "negative vertex id"; return false; }
      for (int b = a + 1; b < 4; ++b)
        if (vid[e * 4 + a] == vid[e * 4 + b]) { *err = "element with repeated vertex id"; return false; }
    }
  std::sort(keys.begin(), keys.end(), [](const Key& x, const Key& y) {
    if (x.a != y.a) return x.a < y.a;
    if (x.b != y.b) return x.b < y.b;
    if (x.c != y.c) return x.c < y.c;
    return x.ef < y.ef;
  });
  auto same = [](const Key& x, const Key& y) { return x.a == y.a && x.b == y.b && x.c == y.c; };
  const size_t nf = keys.size();
  for (size_t k = 0; k < nf; k += 2) {
    if (k + 1 >= nf || !same(keys[k], keys[k + 1]) || (k + 2 < nf && same(keys[k + 1], keys[k + 2]))) {
      *err = "face not matched exactly twice (mesh must be closed/periodic)";
      return false;
    }
  }
  out->nb.assign(nf, -1);
  out->j.assign(nf, 0);
  out->h.assign(nf, 0);
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < static_cast<int64_t>(nf); k += 2) {
    const int64_t f1 = keys[k].ef, f2 = keys[k + 1].ef;
    for (int side = 0; side < 2; ++side) {
      const int64_t me = side ? f2 : f1, ot = side ? f1 : f2;
      const int64_t e = me / 4, n = ot / 4;
      const int i = static_cast<int>(me % 4), jj = static_cast<int>(ot % 4);
      out->nb[me] = n;
      out->j[me] = static_cast<int8_t>(jj);
      const int64_t first = vid[e * 4 + kFaces[i][0]];
      int hh = 0;
      for (int t = 0; t < 3; ++t)
        if (vid[n * 4 + kFaces[jj][t]] == first) hh = t;
      out->h[me] = static_cast<int8_t>(hh);
    }
  }
  for (int64_t e = 0; e < ne; ++e)
    for (int i = 0; i < 4; ++i)
      if (out->nb[e * 4 + i] == e) { *err = "element is its own neighbour (mesh too small)"; return false; }
  return true;
}

bool element_coeffs(int P, int64_t e0, int64_t n, const double* xyz, const double* material,
                    const double* anelastic, const Neighbours& nbr, ElementCoeffs* out,
                    std::string* err) {
  out->star.assign(static_cast<size_t>(n) * 3 * P * 3, 0.0);
  out->aplus.assign(static_cast<size_t>(n) * 4 * P * P, 0.0);
  out->aminus.assign(static_cast<size_t>(n) * 4 * P * P, 0.0);
  if (P == 27) out->src.assign(static_cast<size_t>(n) * P * P, 0.0);
  if (P == 9) out->face.assign(static_cast<size_t>(n) * 4 * kFaceCoeffs, 0.0);
  const double* omega = P == 27 ? anelastic : nullptr;
  const double* Y = P == 27 ? anelastic + 3 : nullptr;
  bool ok = true;
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t t = 0; t < n; ++t) {
    const int64_t e = e0 + t;
    const double* x = xyz + e * 12;
    double J[3][3];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) J[r][c] = x[(c + 1) * 3 + r] - x[r];
    const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                       J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                       J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    if (!(det > 0.0)) {
#pragma omp critical
      { ok = false; *err = "element with det J <= 0"; }
      continue;
    }
    double Ji[3][3];
    Ji[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / det;
    Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
    Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
    Ji[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / det;
    Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
    Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
    Ji[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / det;
    Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
    Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
    // star matrices of the kernels' derivative directions (setup.h kDirT): A*'^c =
    // sum_d kDirTinv[d][c] A*^d, i.e. the rows of kDirTinv^T J^-1 combine the A^d
    double Jd[3][3];
    for (int c = 0; c < 3; ++c)
      for (int d = 0; d < 3; ++d) Jd[c][d] = kDirTinv[0][c] * Ji[0][d] + kDirTinv[1][c] * Ji[1][d] + kDirTinv[2][c] * Ji[2][d];
    const Mat m = material_of(material + e * 3);
    std::vector<double> A(3 * P * P), tmp(P * P), tmp2(P * P), T(P * P), Ti(P * P), G(P * P);
    for (int d = 0; d < 3; ++d) jacobian(P, d, m.rho, m.lam, m.mu, omega, &A[d * P * P]);
    // star matrices at the fixed 3-column pattern
    for (int c = 0; c < 3; ++c)
      for (int p = 0; p < P; ++p) {
        int cols[3];
        star_cols(P, p, cols);
        for (int k = 0; k < 3; ++k) {
          bool dup = false;
          for (int kk = 0; kk < k; ++kk) dup |= cols[kk] == cols[k];
          double v = 0.0;
          if (!dup)
            for (int d = 0; d < 3; ++d) v += Jd[c][d] * A[d * P * P + p * P + cols[k]];
          out->star[((t * 3 + c) * P + p) * 3 + k] = v;
        }
      }
    if (P == 27) {
      double* E = &out->src[t * P * P];
      const double* Ye = Y + e * 6;
      for (int l = 0; l < 3; ++l) {
        const double yl = Ye[l * 2 + 0], ym = Ye[l * 2 + 1];
        for (int s = 0; s < 6; ++s) {
          for (int f = 0; f < 6; ++f) {
            double v = 0.0;
            if (s < 3 && f < 3) v += yl;  // Ylam tr(theta) on normal stresses
            if (s == f) v += 2.0 * ym;    // 2 Ymu theta_ij
            E[s * P + 9 + 6 * l + f] = -v;
          }
          E[(9 + 6 * l + s) * P + 9 + 6 * l + s] = -omega[l];
        }
      }
    }
    // faces
    for (int i = 0; i < 4; ++i) {
      const int a = kFaces[i][0], b = kFaces[i][1], c = kFaces[i][2];
      double e1[3], e2[3], cr[3];
      for (int r = 0; r < 3; ++r) { e1[r] = x[b * 3 + r] - x[a * 3 + r]; e2[r] = x[c * 3 + r] - x[a * 3 + r]; }
      cr[0] = e1[1] * e2[2] - e1[2] * e2[1];
      cr[1] = e1[2] * e2[0] - e1[0] * e2[2];
      cr[2] = e1[0] * e2[1] - e1[1] * e2[0];
      const double twice_area = std::sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
      const double nrm[3] = {cr[0] / twice_area, cr[1] / twice_area, cr[2] / twice_area};
      const double scale = -twice_area / det;  // -2|S_i| / det J
      double R[3][3], Rt[3][3];
      face_frame(nrm, R);
      for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k) Rt[r][k] = R[k][r];
      rotation(P, R, T.data());
      rotation(P, Rt, Ti.data());
      const Mat mo = material_of(material + nbr.nb[e * 4 + i] * 3);
      const double Zpm = std::sqrt(m.rho * (m.lam + 2 * m.mu)), Zsm = std::sqrt(m.rho * m.mu);
      const double Zpp = std::sqrt(mo.rho * (mo.lam + 2 * mo.mu)), Zsp = std::sqrt(mo.rho * mo.mu);
      if (P == 9) {
        double* fc = &out->face[(t * 4 + i) * kFaceCoeffs];
        fc[0] = nrm[0];
        fc[1] = nrm[1];
        fc[2] = nrm[2];
        const double sp = Zpm + Zpp, ss = Zsm + Zsp;
        fc[3] = Zpm / sp;
        fc[4] = Zpm * Zpp / sp;
        fc[5] = 1.0 / sp;
        fc[6] = Zsm / ss;
        fc[7] = Zsm * Zsp / ss;
        fc[8] = 1.0 / ss;
        fc[9] = scale * m.lam;
        fc[10] = scale * m.mu;
        fc[11] = scale / m.rho;
      }
      // Ax(m-) = A[0]
      for (int side = 0; side < 2; ++side) {
        std::fill(G.begin(), G.end(), 0.0);
        const int pairs[3][2] = {{SXX, VU}, {SXY, VV}, {SXZ, VW}};
        for (int pr = 0; pr < 3; ++pr) {
          const int s = pairs[pr][0], v = pairs[pr][1];
          const double Zm = pr == 0 ? Zpm : Zsm, Zp = pr == 0 ? Zpp : Zsp, den = Zm + Zp;
          if (side == 0) {  // G-: coefficients of the local state
            G[v * P + v] = Zm / den;
            G[v * P + s] = -1.0 / den;
            G[s * P + s] = Zp / den;
            G[s * P + v] = -Zm * Zp / den;
          } else {          // G+: coefficients of the neighbour state
            G[v * P + v] = Zp / den;
            G[v * P + s] = 1.0 / den;
            G[s * P + s] = Zm / den;
            G[s * P + v] = Zm * Zp / den;
          }
        }
        if (side == 0) {
          const int others[3] = {SYY, SZZ, SYZ};
          for (int o : others) G[o * P + o] = 1.0;
          for (int o = 9; o < P; ++o) G[o * P + o] = 1.0;
        }
        matmul(P, A.data(), G.data(), tmp.data());   // Ax G
        matmul(P, tmp.data(), Ti.data(), tmp2.data()); // Ax G T^-1
        matmul(P, T.data(), tmp2.data(), tmp.data());  // T Ax G T^-1
        double* dst = (side == 0 ? out->aplus.data() : out->aminus.data()) + (t * 4 + i) * P * P;
        for (int k = 0; k < P * P; ++k) dst[k] = scale * tmp[k];
      }
    }
  }
  return ok;
}

}  // namespace ydg
