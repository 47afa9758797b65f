/* ydg_lina.h -- C ABI of the LinA workload of libydg.so: ADER-DG-SEM for the linearised
 * acoustic equations on a uniform periodic grid of cuboids (arXiv:1903.11521, §"LinA",
 * P:1452-1559; row NEXT-3 of SURVEY §8(f)).
 *
 * The scheme, per element, with a tensor-product nodal basis
 * q_p = Q_xyzp psi_x(x) psi_y(y) psi_z(z) on the N+1 Gauss-Lobatto points per axis:
 *   D^(d+1) = Kt_x D A*^T + Kt_y D B*^T + Kt_z D C*^T,  D^0 = Q          (eq. lina:derivative)
 *   I       = sum_{d=0}^{N} dt^(d+1)/(d+1)! D^d                          (eq. lina:integration)
 *   Q*      = Q + Kh_x I A*^T + Kh_y I B*^T + Kh_z I C*^T
 *   X^s     = F^s I (the side nodes of I),  s in {left, right, bottom, top, back, front}
 *   Q^(n+1) = Q* + sum_s Fh^s (X^s (A+)^sT + X^Neigh(s) (A-)^sT)           (eq. lina3d_flux)
 * with the readings L1-L8 of DESIGN.md §3 (acoustics q = (p, u, v, w); lumped GLL mass
 * matrix; exact Godunov flux with both materials).
 *
 * Conventions: every function returns 0 (YDG_OK) or a YDG_ERR_* code of ydg.h; host
 * pointers are borrowed for the duration of the call; device memory is owned by the handle.
 * DOF layout across the ABI: [element][quantity p][x][y][z] (x slowest), element
 * e = i + nx (j + ny k) for grid cell (i, j, k).  fp64 storage and arithmetic.
 */
#ifndef YDG_LINA_H
#define YDG_LINA_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ydg_lina ydg_lina; /* opaque, owned by the library */

/* N = polynomial degree per axis, 1 <= N <= 7 (order N+1 <= 8: one element's three
 * (N+1)^3 x 4 work tensors fit the shared memory of a CTA); precision must be 8. */
int ydg_lina_create(int order, int precision, int cuda_device, ydg_lina** out);

/* Uniform periodic grid of nx x ny x nz cuboids of size h[3] = (hx, hy, hz) (> 0);
 * material [E][2] = (rho, K) per element (> 0), E = nx ny nz.  Builds the star matrices
 * A*, B*, C* and the Godunov flux solvers (A+-)^s of every side on the host in fp64.
 * DOFs are zero after this call. */
int ydg_lina_upload_grid(ydg_lina* h, int nx, int ny, int nz, const double* hxyz, const double* material);

/* Copy DOFs of elements [first, first+count) from / to host memory (layout above). */
int ydg_lina_upload_dofs(ydg_lina* h, int64_t first, int64_t count, const double* Q);
int ydg_lina_download_dofs(ydg_lina* h, int64_t first, int64_t count, double* Q_out);

/* nsteps time steps of size dt, enqueued on cuda_stream (NULL = the handle's stream): two
 * kernel launches per step (lina_local: ADER predictor, volume, sides; lina_flux). */
int ydg_lina_step(ydg_lina* h, double dt, int nsteps, void* cuda_stream);

/* Scalars: 0 elements, 1 nonzero flops per element-update, 2 algorithmic HBM bytes per
 * element-update, 3 device bytes held, 4 kernel launches per step. */
int ydg_lina_query(ydg_lina* h, int what, double* value);

const char* ydg_lina_error_string(const ydg_lina* h);
void ydg_lina_destroy(ydg_lina* h);

#ifdef __cplusplus
}
#endif
#endif /* YDG_LINA_H */
