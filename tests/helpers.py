"""Shared test helpers: run the library through its C ABI and the oracle on the same inputs."""
import numpy as np

import synth
from oracle import step as ostep


def make_inputs(cfg):
    xyz, vid = synth.kuhn_mesh(cfg.nx, cfg.ny, cfg.nz, seed=cfg.seed, jitter=cfg.jitter)
    mat = synth.material(cfg)
    Q = synth.dofs(cfg)
    an = None
    if cfg.P == 27:
        omega, Y = synth.anelastic(cfg, mat)
        an = np.concatenate([omega, Y.ravel()])
    return xyz, vid, mat, Q, an


LAST_PATH = {}  # kernel path (ydg_query YDG_Q_KERNEL_PATH) of the last run_gpu call


def run_gpu(cfg, xyz, vid, mat, Q, an=None, nsteps=None, dt=None):
    import paper_1903_11521_b200 as ydg
    h = ydg.ydg_create(cfg.N, cfg.P, cfg.precision)
    ydg.ydg_upload_mesh(h, xyz, vid, mat, an)
    LAST_PATH["path"] = int(ydg.ydg_query(h, ydg.YDG_Q_KERNEL_PATH))
    ydg.ydg_upload_dofs(h, 0, Q.astype(h.dtype))
    ydg.ydg_step(h, cfg.dt if dt is None else dt, cfg.steps if nsteps is None else nsteps)
    out = ydg.ydg_download_dofs(h, 0, Q.shape[0])
    nbt = ydg.ydg_get_neighbours(h, 0, Q.shape[0])
    ydg.ydg_destroy(h)
    return out.astype(np.float64), nbt


def run_oracle(cfg, xyz, vid, mat, Q, an=None, nsteps=None, dt=None):
    omega = Y = None
    if cfg.P == 27:
        omega = an[:3]
        Y = an[3:].reshape(-1, 3, 2)
    prob = ostep.setup(cfg.N, xyz, vid, mat, P=cfg.P, omega=omega, Y=Y)
    Qi = ostep.to_internal(Q.astype(np.float64))
    out = ostep.step(prob, Qi, cfg.dt if dt is None else dt, cfg.steps if nsteps is None else nsteps)
    return ostep.to_canonical(out)


def rel_err(got, ref):
    """max |got - ref| / max |ref| (BASELINE north_star metric), plus per quantity group."""
    d = np.abs(got - ref)
    out = {"all": d.max() / np.abs(ref).max()}
    groups = {"stress": slice(0, 6), "velocity": slice(6, 9), "memory": slice(9, None)}
    for g, s in groups.items():
        r = ref[:, s]
        if r.size and np.abs(r).max() > 0:
            out[g] = d[:, s].max() / np.abs(r).max()
    return out
