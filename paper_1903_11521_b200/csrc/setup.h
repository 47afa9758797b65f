// Host-side setup of the ADER-DG element update: mesh validation, face matching,
// geometry, star matrices and Godunov flux solvers (fp64).  Shares no code with the test oracle.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace ydg {

// local faces as outward-oriented vertex triples (reading R7)
constexpr int kFaces[4][3] = {{0, 2, 1}, {0, 1, 3}, {0, 3, 2}, {1, 2, 3}};

struct Neighbours {
  std::vector<int64_t> nb;  // [ne][4] Neigh
  std::vector<int8_t> j;    // [ne][4] Face
  std::vector<int8_t> h;    // [ne][4] Rot
};

// Match faces by sorted vertex-id triples.  Returns false and sets err on a mesh error.
bool match_faces(int64_t ne, const int64_t* vid, Neighbours* out, std::string* err);

struct ElementCoeffs {
  // per element, fp64, for P quantities:
  //  star: [3][P][3] values of A*^c at the fixed 3-column pattern of row p (star_cols)
  //  aplus / aminus: [4][P][P] flux solvers with -2|S_i|/det J folded in (row-major p,q)
  //  src: [P][P] viscoelastic source E (P = 27 only)
  //  face: [4][kFaceCoeffs] factored flux solver of face i (P = 9; see kFaceCoeffs)
  std::vector<double> star, aplus, aminus, src, face;
};

// Factored form of the elastic flux solvers of one face (reading R8), all scaled by
// s = -2|S_i|/det J:  n (3), then per wave type w in {p, s}: Z-/(Z-+Z+), Z-Z+/(Z-+Z+),
// 1/(Z-+Z+), then s*lambda-, s*mu-, s/rho-.  A+ q- + A- q+ = the flux of the Godunov state
// built from these (dm_flux).
constexpr int kFaceCoeffs = 12;

// Derivative directions of the CK and volume products ("sparser derivative
// directions"): the kernels use K'^c = sum_d kDirT[c][d] K^d (reference directions (1,0,0),
// (0,1,-1), (1,-2,0) of the Dubiner basis: 924 instead of 1,708 nonzeros at N = 5) with the
// star matrices A*'^c = sum_d kDirTinv[d][c] A*^d, so that sum_c K'^c X A*'^c = sum_c K^c X
// A*^c exactly (P:1312-1340 unchanged up to rounding).  Keep in sync with gen/tables.py KDIR_T.
constexpr double kDirT[3][3] = {{1, 0, 0}, {0, 1, -1}, {1, -2, 0}};
constexpr double kDirTinv[3][3] = {{1, 0, 0}, {0.5, 0, -0.5}, {0.5, -1, -0.5}};
// K'^c[k][l] from the reference matrices K (exact cancellations -> exact zeros)
template <class KA>
inline double kdir(const KA& K, int c, int k, int l) {
  double v = 0.0, m = 0.0;
  for (int d = 0; d < 3; ++d) {
    v += kDirT[c][d] * K[d][k][l];
    m = m > (K[d][k][l] < 0 ? -K[d][k][l] : K[d][k][l]) ? m : (K[d][k][l] < 0 ? -K[d][k][l] : K[d][k][l]);
  }
  return (v < 0 ? -v : v) <= 1e-12 * m ? 0.0 : v;
}

// Columns of the star-matrix pattern of row p (3 per row; unused slots repeat a column
// with a zero coefficient).  Valid for P = 9 and P = 27.
void star_cols(int P, int p, int cols[3]);

// Compute coefficients for elements [e0, e0+n) of the global mesh.
//  anelastic: NULL or [3] omega then [ne][3][2] (Ylam, Ymu).
bool element_coeffs(int P, int64_t e0, int64_t n, const double* xyz, const double* material,
                    const double* anelastic, const Neighbours& nbr, ElementCoeffs* out,
                    std::string* err);

}  // namespace ydg
