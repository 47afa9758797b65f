"""B200-native ADER-DG element update (arXiv:1903.11521 Sec. 5.1) -- Python binding.

Thin ctypes marshalling over the C ABI of ``libydg.so`` (declared in ``include/ydg.h``);
every step of the method runs in the library's CUDA kernels.  There is no CPU fallback:
importing works without a GPU (so the ABI can be inspected), but any compute call on a
machine without the built library or a CUDA device raises.

    import paper_1903_11521_b200 as ydg
    h = ydg.ydg_create(5, 9, 8)
    ydg.ydg_upload_mesh(h, xyz, vid, material)
    ydg.ydg_upload_dofs(h, 0, Q)            # canonical [element][quantity][basis]
    ydg.ydg_step(h, dt, 10)
    Q1 = ydg.ydg_download_dofs(h, 0, n)
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("YDG_LIB") or os.path.join(_HERE, "libydg.so")

YDG_OK, YDG_ERR_ARG, YDG_ERR_STATE, YDG_ERR_CUDA, YDG_ERR_NCCL, YDG_ERR_MESH, YDG_ERR_OOM, \
    YDG_ERR_UNSUPPORTED = range(8)
(YDG_Q_N_ELEMENTS, YDG_Q_FIRST_LOCAL, YDG_Q_N_LOCAL, YDG_Q_NZ_FLOPS, YDG_Q_ALG_BYTES, YDG_Q_B,
 YDG_Q_BTILDE, YDG_Q_DEVICE_BYTES, YDG_Q_LAUNCHES_PER_STEP, YDG_Q_LOCAL_BYTES, YDG_Q_NEIGH_BYTES,
 YDG_Q_LOCAL_FLOPS, YDG_Q_NEIGH_FLOPS, YDG_Q_PROF_LOCAL_MS, YDG_Q_PROF_NEIGH_MS,
 YDG_Q_PROF_LAUNCHES, YDG_Q_KERNEL_PATH, YDG_Q_SIMULATIONS, YDG_Q_TILE_ELEMENTS,
 YDG_Q_NEIGH_FLOPS_EXEC, YDG_Q_GUARD_VIOLATIONS, YDG_Q_MAX_ABS_Q, YDG_Q_FUSED, YDG_Q_PROF_FUSED_MS,
 YDG_Q_FUSED_BYTES) = range(25)

EXPORTS = ("ydg_create", "ydg_last_error", "ydg_set_comm", "ydg_set_simulations", "ydg_upload_mesh", "ydg_upload_dofs",
           "ydg_upload_dofs_device", "ydg_download_dofs_device", "ydg_step", "ydg_step_graph", "ydg_set_clusters", "ydg_step_lts", "ydg_synchronize",
           "ydg_download_dofs", "ydg_get_neighbours", "ydg_halo_plan", "ydg_profile", "ydg_query",
           "ydg_error_string", "ydg_destroy",
           # LinA workload (include/ydg_lina.h)
           "ydg_lina_create", "ydg_lina_upload_grid", "ydg_lina_upload_dofs", "ydg_lina_download_dofs",
           "ydg_lina_step", "ydg_lina_query", "ydg_lina_error_string", "ydg_lina_destroy")


class YdgError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"ydg error {code}: {msg}")
        self.code = code


_lib = None


def lib():
    """Load libydg.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run python -m paper_1903_11521_b200.build")
        L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.ydg_create.argtypes = [i32, i32, i32, i32, ctypes.POINTER(vp)]
        L.ydg_last_error.restype = ctypes.c_char_p
        L.ydg_set_comm.argtypes = [vp, i32, i32, ctypes.c_char_p]
        L.ydg_upload_mesh.argtypes = [vp, i64, vp, vp, vp, vp]
        L.ydg_set_simulations.argtypes = [vp, i32]
        L.ydg_upload_dofs.argtypes = [vp, i64, i64, vp]
        L.ydg_upload_dofs_device.argtypes = [vp, i64, i64, vp, vp]
        L.ydg_download_dofs_device.argtypes = [vp, i64, i64, vp, vp]
        L.ydg_step.argtypes = [vp, dbl, i32, vp]
        L.ydg_step_graph.argtypes = [vp, dbl, i32, vp]
        L.ydg_set_clusters.argtypes = [vp, vp, i64]
        L.ydg_step_lts.argtypes = [vp, dbl, i32, vp]
        L.ydg_synchronize.argtypes = [vp]
        L.ydg_download_dofs.argtypes = [vp, i64, i64, vp]
        L.ydg_get_neighbours.argtypes = [vp, i64, i64, vp, vp, vp]
        L.ydg_profile.argtypes = [vp, i32]
        L.ydg_halo_plan.argtypes = [i64, vp, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.ydg_query.argtypes = [vp, i32, ctypes.POINTER(dbl)]
        L.ydg_error_string.argtypes = [vp]
        L.ydg_error_string.restype = ctypes.c_char_p
        L.ydg_destroy.argtypes = [vp]
        L.ydg_destroy.restype = None
        L.ydg_lina_create.argtypes = [i32, i32, i32, ctypes.POINTER(vp)]
        L.ydg_lina_upload_grid.argtypes = [vp, i32, i32, i32, vp, vp]
        L.ydg_lina_upload_dofs.argtypes = [vp, i64, i64, vp]
        L.ydg_lina_download_dofs.argtypes = [vp, i64, i64, vp]
        L.ydg_lina_step.argtypes = [vp, dbl, i32, vp]
        L.ydg_lina_query.argtypes = [vp, i32, ctypes.POINTER(dbl)]
        L.ydg_lina_error_string.argtypes = [vp]
        L.ydg_lina_error_string.restype = ctypes.c_char_p
        L.ydg_lina_destroy.argtypes = [vp]
        L.ydg_lina_destroy.restype = None
        _lib = L
    return _lib


class Handle:
    """Owns a ydg_solver*; remembers order / quantities / precision for marshalling."""

    def __init__(self, ptr, order, quantities, precision):
        self.ptr, self.N, self.P, self.precision = ptr, order, quantities, precision
        self.B = (order + 1) * (order + 2) * (order + 3) // 6
        self.dtype = np.float64 if precision == 8 else np.float32

    def __del__(self):
        if getattr(self, "ptr", None):
            ydg_destroy(self)


def _check(h, rc):
    if rc != YDG_OK:
        raise YdgError(rc, lib().ydg_error_string(h.ptr).decode())


def _c(a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a, a.ctypes.data_as(ctypes.c_void_p)


def ydg_create(order, quantities=9, precision=8, device=0):
    out = ctypes.c_void_p()
    rc = lib().ydg_create(order, quantities, precision, device, ctypes.byref(out))
    if rc != YDG_OK:
        raise YdgError(rc, lib().ydg_last_error().decode())
    return Handle(out.value, order, quantities, precision)


def ydg_set_comm(h, rank, nranks, nccl_unique_id: bytes):
    _check(h, lib().ydg_set_comm(h.ptr, rank, nranks, nccl_unique_id))


def ydg_set_simulations(h, S):
    _check(h, lib().ydg_set_simulations(h.ptr, int(S)))


def ydg_upload_mesh(h, elem_xyz, elem_vid, material, anelastic=None):
    xyz, pxyz = _c(elem_xyz, np.float64)
    vid, pvid = _c(elem_vid, np.int64)
    mat, pmat = _c(material, np.float64)
    ne = xyz.shape[0] if xyz.ndim else 0
    if xyz.shape != (ne, 4, 3) or vid.shape != (ne, 4) or mat.shape != (ne, 3):
        raise ValueError(f"mesh shapes: xyz {xyz.shape} (want (ne,4,3)), vid {vid.shape} (ne,4), "
                         f"material {mat.shape} (ne,3)")
    if anelastic is not None:
        an, pan = _c(anelastic, np.float64)
        if an.size != 3 + 6 * ne:
            raise ValueError(f"anelastic: {an.size} values, want 3 + 6 ne = {3 + 6 * ne}")
    else:
        an, pan = None, None
    _check(h, lib().ydg_upload_mesh(h.ptr, xyz.shape[0], pxyz, pvid, pmat, pan))


def ydg_upload_dofs(h, first, Q):
    q, pq = _c(Q, h.dtype)
    if q.ndim != 3 or q.shape[1:] != (h.P, h.B):
        raise ValueError(f"Q shape {q.shape}, want (count, P={h.P}, B={h.B})")
    _check(h, lib().ydg_upload_dofs(h.ptr, first, q.shape[0], pq))


def ydg_upload_dofs_device(h, first, count, ptr, stream=None):
    _check(h, lib().ydg_upload_dofs_device(h.ptr, first, count, ctypes.c_void_p(ptr), ctypes.c_void_p(stream)))


def ydg_download_dofs_device(h, first, count, ptr, stream=None):
    _check(h, lib().ydg_download_dofs_device(h.ptr, first, count, ctypes.c_void_p(ptr), ctypes.c_void_p(stream)))


def ydg_step(h, dt, nsteps=1, stream=None):
    _check(h, lib().ydg_step(h.ptr, float(dt), int(nsteps), ctypes.c_void_p(stream)))


def ydg_step_graph(h, dt, nsteps=1, stream=None):
    _check(h, lib().ydg_step_graph(h.ptr, float(dt), int(nsteps), ctypes.c_void_p(stream)))


def ydg_set_clusters(h, cluster):
    c, pc = _c(cluster, np.int8)
    _check(h, lib().ydg_set_clusters(h.ptr, pc, c.size))


def ydg_step_lts(h, dt, ncycles=1, stream=None):
    _check(h, lib().ydg_step_lts(h.ptr, float(dt), int(ncycles), ctypes.c_void_p(stream)))


def ydg_synchronize(h):
    _check(h, lib().ydg_synchronize(h.ptr))


def ydg_download_dofs(h, first, count, out=None):
    if out is None:
        out = np.empty((count, h.P, h.B), dtype=h.dtype)
    assert out.dtype == h.dtype and out.flags.c_contiguous and out.shape == (count, h.P, h.B)
    _check(h, lib().ydg_download_dofs(h.ptr, first, count, out.ctypes.data_as(ctypes.c_void_p)))
    return out


def ydg_get_neighbours(h, first, count):
    nb = np.empty((count, 4), dtype=np.int64)
    j = np.empty((count, 4), dtype=np.int8)
    hr = np.empty((count, 4), dtype=np.int8)
    _check(h, lib().ydg_get_neighbours(h.ptr, first, count, nb.ctypes.data_as(ctypes.c_void_p),
                                       j.ctypes.data_as(ctypes.c_void_p), hr.ctypes.data_as(ctypes.c_void_p)))
    return nb, j, hr


def ydg_halo_plan(elem_vid, rank, nranks):
    """Host-only: the z-slab halo plan of `rank` (dict of numpy arrays); no GPU needed."""
    vid, pvid = _c(elem_vid, np.int64)
    counts = np.zeros(3, dtype=np.int64)
    P = ctypes.c_void_p
    rc = lib().ydg_halo_plan(vid.shape[0], pvid, rank, nranks, counts.ctypes.data_as(P), None, None, None,
                             None, None, None, None, None)
    if rc != YDG_OK:
        raise YdgError(rc, lib().ydg_last_error().decode())
    npeer, ng, ns = (int(x) for x in counts)
    peers = np.zeros(npeer, dtype=np.int32)
    rcnt = np.zeros(npeer, dtype=np.int64)
    scnt = np.zeros(npeer, dtype=np.int64)
    ghost = np.zeros(ng, dtype=np.int64)
    send = np.zeros(ns, dtype=np.int64)
    sface = np.zeros(ns, dtype=np.int8)
    recv = np.zeros(ns, dtype=np.int64)
    rface = np.zeros(ns, dtype=np.int8)
    rc = lib().ydg_halo_plan(vid.shape[0], pvid, rank, nranks, counts.ctypes.data_as(P), peers.ctypes.data_as(P),
                             rcnt.ctypes.data_as(P), scnt.ctypes.data_as(P), ghost.ctypes.data_as(P),
                             send.ctypes.data_as(P), sface.ctypes.data_as(P), recv.ctypes.data_as(P),
                             rface.ctypes.data_as(P))
    if rc != YDG_OK:
        raise YdgError(rc, lib().ydg_last_error().decode())
    return {"peers": peers, "recv_cnt": rcnt, "send_cnt": scnt, "ghost_of": ghost, "send_elem": send,
            "send_face": sface, "recv_elem": recv, "recv_face": rface}


def ydg_profile(h, enable=True):
    _check(h, lib().ydg_profile(h.ptr, 1 if enable else 0))


def ydg_query(h, what):
    v = ctypes.c_double()
    _check(h, lib().ydg_query(h.ptr, what, ctypes.byref(v)))
    return v.value


def ydg_destroy(h):
    if h.ptr:
        lib().ydg_destroy(h.ptr)
        h.ptr = None


# ---------------------------------------------------------------- LinA (include/ydg_lina.h)

LINA_Q_ELEMENTS, LINA_Q_NZ_FLOPS, LINA_Q_ALG_BYTES, LINA_Q_DEVICE_BYTES, LINA_Q_LAUNCHES = range(5)


class LinaHandle:
    """Owns a ydg_lina*: ADER-DG-SEM acoustics on a uniform periodic cuboid grid."""

    def __init__(self, ptr, order):
        self.ptr, self.N = ptr, order
        self.n = order + 1
        self.E = 0

    def __del__(self):
        if getattr(self, "ptr", None):
            lina_destroy(self)


def _lcheck(h, rc):
    if rc != YDG_OK:
        raise YdgError(rc, lib().ydg_lina_error_string(h.ptr).decode())


def lina_create(order, precision=8, device=0):
    out = ctypes.c_void_p()
    rc = lib().ydg_lina_create(order, precision, device, ctypes.byref(out))
    if rc != YDG_OK:
        raise YdgError(rc, "ydg_lina_create")
    return LinaHandle(out.value, order)


def lina_upload_grid(h, nx, ny, nz, hxyz, material):
    hh, ph = _c(hxyz, np.float64)
    m, pm = _c(material, np.float64)
    if hh.shape != (3,) or m.shape != (nx * ny * nz, 2):
        raise ValueError(f"h {hh.shape} (want (3,)), material {m.shape} (want ({nx * ny * nz}, 2))")
    _lcheck(h, lib().ydg_lina_upload_grid(h.ptr, nx, ny, nz, ph, pm))
    h.E = nx * ny * nz


def lina_upload_dofs(h, first, Q):
    q, pq = _c(Q, np.float64)
    n = h.n
    if q.ndim != 5 or q.shape[1:] != (4, n, n, n):
        raise ValueError(f"Q shape {q.shape}, want (count, 4, {n}, {n}, {n})")
    _lcheck(h, lib().ydg_lina_upload_dofs(h.ptr, first, q.shape[0], pq))


def lina_download_dofs(h, first, count):
    n = h.n
    out = np.empty((count, 4, n, n, n), dtype=np.float64)
    _lcheck(h, lib().ydg_lina_download_dofs(h.ptr, first, count, out.ctypes.data_as(ctypes.c_void_p)))
    return out


def lina_step(h, dt, nsteps=1, stream=None):
    _lcheck(h, lib().ydg_lina_step(h.ptr, float(dt), int(nsteps), ctypes.c_void_p(stream)))


def lina_query(h, what):
    v = ctypes.c_double()
    _lcheck(h, lib().ydg_lina_query(h.ptr, what, ctypes.byref(v)))
    return v.value


def lina_destroy(h):
    if h.ptr:
        lib().ydg_lina_destroy(h.ptr)
        h.ptr = None
