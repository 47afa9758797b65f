/* ydg.h -- C ABI of the B200 ADER-DG element-update library (libydg.so).
 *
 * Implements the element-local ADER-DG update of the elastic (and viscoelastic) wave
 * equation on tetrahedra, arXiv:1903.11521 (Uphoff & Bader) Sec. 5.1, Eqs.
 * (seissol:derivative) P:1312-1317, (seissol:timeint) P:1326-1333,
 * (seissol:correction_local) P:1334-1341 and (seissol:correction_neigh) P:1342.
 * "P:n" = line n of the paper source.  Readings where the paper is silent or garbled
 * (basis, face conventions, Riemann solver, viscoelastic equations ...) are in DESIGN.md §3.
 *
 * Conventions
 *  - Every function returns an int status: YDG_OK (0) or one of the error codes below.
 *    ydg_error_string(h) returns the last message of handle h (owned by h, valid until
 *    the next call on h).  A failed call leaves the previous state intact, except CUDA /
 *    NCCL faults, which poison the handle: every later call returns the same error.
 *  - Host pointers are borrowed for the duration of the call only (data is copied).
 *    Device memory is owned by the handle and released by ydg_destroy.
 *  - Canonical DOF layout across the ABI: Q[element][quantity][basis] (the paper's
 *    Q_kp, column-major B x P per element), in the solver precision
 *    (double for precision 8, float for precision 4).  Quantity order:
 *    (sxx, syy, szz, sxy, syz, sxz, u, v, w) then theta^l_(xx,yy,zz,xy,yz,xz), l = 0..2.
 *    Basis order: Dubiner functions by degree, then r, then q (reading R6).
 *  - A handle is not thread-safe.
 */
#ifndef YDG_H
#define YDG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  YDG_OK = 0,
  YDG_ERR_ARG = 1,         /* null pointer, bad size or enum value                         */
  YDG_ERR_STATE = 2,       /* call out of order (e.g. step before mesh upload)            */
  YDG_ERR_CUDA = 3,        /* CUDA runtime error (poisons the handle)                     */
  YDG_ERR_NCCL = 4,        /* NCCL error (poisons the handle)                             */
  YDG_ERR_MESH = 5,        /* face matched != 2 times, det J <= 0, bad vertex ids         */
  YDG_ERR_OOM = 6,         /* device allocation failed                                    */
  YDG_ERR_UNSUPPORTED = 7  /* order / quantities / precision combination not compiled     */
};

/* ydg_query keys */
enum {
  YDG_Q_N_ELEMENTS = 0,        /* global element count                                     */
  YDG_Q_FIRST_LOCAL = 1,       /* first global element id owned by this rank               */
  YDG_Q_N_LOCAL = 2,           /* number of elements owned by this rank                    */
  YDG_Q_NZ_FLOPS = 3,          /* nonzero flops per element-update (executed formulation)  */
  YDG_Q_ALG_BYTES = 4,         /* algorithmic HBM bytes per element-update (both kernels)  */
  YDG_Q_B = 5,                 /* basis functions per element, C(N+3,3)                    */
  YDG_Q_BTILDE = 6,            /* face basis functions, C(N+2,2)                           */
  YDG_Q_DEVICE_BYTES = 7,      /* device memory held by the handle                         */
  YDG_Q_LAUNCHES_PER_STEP = 8, /* kernel launches of one ydg_step(nsteps = 1)              */
  YDG_Q_LOCAL_BYTES = 9,       /* algorithmic bytes / element of the local kernel          */
  YDG_Q_NEIGH_BYTES = 10,      /* algorithmic bytes / element of the neighbour kernel      */
  YDG_Q_LOCAL_FLOPS = 11,      /* nonzero flops / element of the local kernel              */
  YDG_Q_NEIGH_FLOPS = 12,      /* nonzero flops / element of the neighbour kernel          */
  YDG_Q_PROF_LOCAL_MS = 13,    /* profiling: summed device time of local-kernel launches   */
  YDG_Q_PROF_NEIGH_MS = 14,    /* profiling: summed device time of neighbour launches      */
  YDG_Q_PROF_LAUNCHES = 15,    /* profiling: number of timed kernel launches               */
  YDG_Q_KERNEL_PATH = 16,      /* kernels a step runs: 0 fp64 elastic tensor-core (dm_local/
                                  dm_flux), 1 fp32 sparse FFMA (ader_*), 2 viscoelastic
                                  tensor-core (vm_local/vm_neigh), 3 generic CSR (gen_*)    */
  YDG_Q_SIMULATIONS = 17,      /* fused simulations S (ydg_set_simulations)                 */
  YDG_Q_TILE_ELEMENTS = 18,    /* elements per tile of the tiled kernels (8 fp64, 32 fp32)  */
  YDG_Q_NEIGH_FLOPS_EXEC = 19, /* nonzero flops / element the neighbour kernel executes (the
                                  fp64 flux kernel lifts local + neighbour flux once per face;
                                  YDG_Q_NEIGH_FLOPS counts the canonical two lifts)           */
  YDG_Q_GUARD_VIOLATIONS = 20, /* debug: with YDG_GUARD=1 in the environment at ydg_create,
                                  every device buffer of the mesh and DOFs has 64 KiB guard
                                  zones of a fill pattern on both sides; this query
                                  synchronises the device and returns the number of guard
                                  bytes overwritten (0 = no out-of-bounds store seen), -1 when
                                  the handle has no guards, -2 on a CUDA error              */
  YDG_Q_MAX_ABS_Q = 21,        /* diagnostic: max |Q| over the owned DOFs (a reduction
                                  kernel on the handle's stream, synchronised); NaN when any
                                  DOF is NaN or infinite                                     */
  YDG_Q_FUSED = 22,            /* 1 when ydg_step(nsteps >= 2) runs the fused step kernel
                                  (opt-in: YDG_FUSED=1 in the environment at mesh upload;
                                  fp64 elastic tensor-core path, one rank, room for a second
                                  trace buffer), else 0                                      */
  YDG_Q_PROF_FUSED_MS = 23,    /* profiling: summed device time of fused-kernel launches    */
  YDG_Q_FUSED_BYTES = 24       /* algorithmic bytes / element of the fused kernel (Q read
                                  and written once; traces written, own + neighbour read)    */
};

typedef struct ydg_solver ydg_solver; /* opaque, owned by the library */

/* Create a solver.
 *  order      N = maximum polynomial degree (B = C(N+3,3)); compiled: 1..6.
 *  quantities 9 = elastic, 27 = viscoelastic with 3 mechanisms.
 *  precision  8 = fp64, 4 = fp32 (storage and arithmetic; setup is fp64, rounded once).
 *  cuda_device  device ordinal used by every later call.
 *  out        receives the handle; *out = NULL on failure (then use ydg_last_error()). */
int ydg_create(int order, int quantities, int precision, int cuda_device, ydg_solver** out);

/* Static message of the last ydg_create failure (thread-local). */
const char* ydg_last_error(void);

/* Optional, before ydg_upload_mesh: join a z-slab decomposition over nranks GPUs.
 *  nccl_unique_id  128 bytes from ncclGetUniqueId on rank 0 (same on all ranks).
 *  Rank r owns global elements [r*ne/nranks, (r+1)*ne/nranks) (the generator orders
 *  elements z-major, so ranges are slabs).  NCCL is loaded at run time (libnccl.so.2). */
int ydg_set_comm(ydg_solver* h, int rank, int nranks, const void* nccl_unique_id);
/*  A unique id whose first 7 bytes are "YDGLOOP" selects the loopback transport instead of
 *  NCCL: the ranks are handles of one process (one host thread each) on one GPU, the halo
 *  goes device-to-device at host barriers -- for checking partition invariance on a single
 *  GPU; same plan, pack and unpack as the NCCL path. */

/* Optional, before ydg_upload_mesh: S >= 1 fused simulations (an extra index
 * s on the degrees of freedom, Q_skp; the mesh, material, star matrices and flux solvers
 * are shared).  The S simulations of element e are the "element-simulations" v = e*S + s:
 * after ydg_upload_mesh every element id of the DOF calls, ydg_get_neighbours and the
 * YDG_Q_N_ELEMENTS / FIRST_LOCAL / N_LOCAL queries counts element-simulations, so the
 * canonical DOF layout becomes [element][simulation][quantity][basis] and the neighbour of
 * v across face i is Neigh(e, i) * S + s.  On the GPU the simulations of an element are
 * adjacent lanes of a tile (the batch dimension every kernel already vectorises over).
 * S in [1, 64]; YDG_ERR_STATE after ydg_upload_mesh. */
int ydg_set_simulations(ydg_solver* h, int S);

/* Upload the (global) mesh and material; builds geometry, star matrices, flux solvers and
 * the neighbour relation (Neigh, Face, Rot of P:1342) on the host in fp64.
 *  n_elements  global element count (> 0).
 *  elem_xyz    [ne][4][3] vertex coordinates (unwrapped per element; det J > 0 required).
 *  elem_vid    [ne][4] topological vertex ids (periodic ids allowed); faces are matched by
 *              sorted id triples and every face must match exactly twice (YDG_ERR_MESH).
 *  material    [ne][3] = rho, vp, vs (SI units).
 *  anelastic   quantities == 27: [3] omega_l (rad/s), then [ne][3][2] (Ylam_l, Ymu_l);
 *              otherwise NULL.
 * DOFs are zero after this call. */
int ydg_upload_mesh(ydg_solver* h, int64_t n_elements, const double* elem_xyz,
                    const int64_t* elem_vid, const double* material, const double* anelastic);

/* Copy DOFs of global elements [first, first+count) (must be owned by this rank) from
 * host memory Q (canonical layout, solver precision) to the device.  Pinned memory is
 * used asynchronously on `cuda_stream` when ydg_step follows on the same stream. */
int ydg_upload_dofs(ydg_solver* h, int64_t first, int64_t count, const void* Q);

/* Same as ydg_upload_dofs / ydg_download_dofs with a device pointer in canonical layout
 * (no host copy), enqueued on cuda_stream (NULL = the handle's stream). */
int ydg_upload_dofs_device(ydg_solver* h, int64_t first, int64_t count, const void* Q_dev,
                           void* cuda_stream);
int ydg_download_dofs_device(ydg_solver* h, int64_t first, int64_t count, void* Q_dev,
                             void* cuda_stream);

/* Advance all owned elements by nsteps global time steps of size dt.
 * Enqueued on cuda_stream (NULL = the handle's own stream); returns without waiting.
 * Collective over the ranks of ydg_set_comm: all must call with the same dt, nsteps.
 * Launches: two per step (local part, flux); with YDG_Q_FUSED = 1 and nsteps >= 2,
 * nsteps + 1: the local part of step 0, nsteps - 1 fused kernels (flux of step n - 1, then
 * the local part of step n, per tile; the traces alternate between two buffers) and the
 * flux of the last step.  Either way Q holds the complete state when the call's work ends. */
int ydg_step(ydg_solver* h, double dt, int nsteps, void* cuda_stream);

/* Same as ydg_step, launched as one CUDA graph: the 2 * nsteps kernel launches of (dt,
 * nsteps) are captured on first use (and again whenever dt or nsteps change or a mesh is
 * uploaded) and replayed with one cudaGraphLaunch on cuda_stream -- for small meshes whose
 * steps are launch-latency bound (BASELINE configs[0]: 384 elements).  One rank only
 * (YDG_ERR_UNSUPPORTED otherwise); profiling must be off (YDG_ERR_STATE). */
int ydg_step_graph(ydg_solver* h, double dt, int nsteps, void* cuda_stream);

/* Optional, before ydg_upload_mesh: two-cluster local time stepping (the paper's LTS of
 * Table loh1; scheme = reading R26 of DESIGN.md, rate 2).  cluster[n] per
 * element (caller numbering): 0 advances by dt, 1 by 2 dt.  The number of 1s must be a
 * multiple of YDG_Q_TILE_ELEMENTS (every launch covers whole tiles of one cluster).  fp64
 * elastic tensor-core path on one rank (YDG_ERR_UNSUPPORTED otherwise, at upload). */
int ydg_set_clusters(ydg_solver* h, const int8_t* cluster, int64_t n);

/* One LTS cycle takes every element from t to t + 2 dt: coarse sub-interval traces, coarse
 * local update (2 dt), two fine substeps (local + flux with the coarse neighbours' traces of
 * the matching half interval), then the coarse flux with the sum of the fine substeps'
 * traces.  ncycles cycles, enqueued on cuda_stream (NULL = the handle's stream). */
int ydg_step_lts(ydg_solver* h, double dt, int ncycles, void* cuda_stream);

/* Block until all work of the handle has finished. */
int ydg_synchronize(ydg_solver* h);

/* Copy DOFs of owned elements [first, first+count) to host memory Q_out (canonical
 * layout, solver precision).  Blocking. */
int ydg_download_dofs(ydg_solver* h, int64_t first, int64_t count, void* Q_out);

/* Neighbour relation of owned elements [first, first+count): nb [count][4] global element
 * ids (Neigh), j [count][4] neighbour local face (Face), hrot [count][4] orientation (Rot,
 * position of the element's face-first vertex id in the neighbour's face triple), with
 * local faces (0,2,1), (0,1,3), (0,3,2), (1,2,3) (reading R7). */
int ydg_get_neighbours(ydg_solver* h, int64_t first, int64_t count, int64_t* nb, int8_t* j,
                       int8_t* hrot);

/* Enable (1) / disable (0) per-launch CUDA-event timing of the element kernels inside
 * ydg_step (events recorded on the launch stream around every launch).  Enabling resets
 * the totals; ydg_query(YDG_Q_PROF_*) synchronises with the recorded events. */
int ydg_profile(ydg_solver* h, int enable);

/* Host-only helper (no device needed): the z-slab halo plan ydg_set_comm + ydg_upload_mesh
 * would build for `rank` of `nranks` on the mesh given by elem_vid [ne][4].  The halo
 * moves one face block (the time-integrated trace of one side of a face, Bt x P values)
 * per face whose two elements live on different ranks (the neighbour flux reads
 * the neighbour's trace on the shared face only).
 *  counts[3] <- (number of peers np, number of ghost elements ng, number of face blocks nb
 *              sent = received).
 *  If the array arguments are non-NULL they must hold counts[] entries and receive:
 *  peers[np] (ascending), recv_cnt[np], send_cnt[np] (face blocks per peer, equal),
 *  ghost_of[ng] (global ids of the ghost slots, grouped by peer, ascending within a peer),
 *  send_elem[nb] / send_face[nb] (global id and local face of every block sent, grouped by
 *  peer, ordered by (id, face)) and recv_elem[nb] / recv_face[nb] (the sending element's
 *  global id and local face of every block received, same order) -- a peer's send list
 *  equals our receive list from it. */
int ydg_halo_plan(int64_t n_elements, const int64_t* elem_vid, int rank, int nranks,
                  int64_t* counts, int32_t* peers, int64_t* recv_cnt, int64_t* send_cnt,
                  int64_t* ghost_of, int64_t* send_elem, int8_t* send_face, int64_t* recv_elem,
                  int8_t* recv_face);

/* Query a scalar (see YDG_Q_*). */
int ydg_query(ydg_solver* h, int what, double* value);

const char* ydg_error_string(const ydg_solver* h);

/* Release the handle and all its device memory (NULL is a no-op). */
void ydg_destroy(ydg_solver* h);

#ifdef __cplusplus
}
#endif
#endif /* YDG_H */
