#!/usr/bin/env python
"""Benchmark of the B200 ADER-DG element update (arXiv:1903.11521 Sec. 5.1).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1] [--impl ydg|reference]

One *step* = one global ADER-DG time step of every element of the workload (the whole hot
path: CK recursion, time integral, volume, local and neighbour flux = BASELINE.json
north_star), i.e. one ``ydg_step(dt, 1)`` call = two kernel launches.  Metric: element-
updates/s (plus nonzero GFLOP/s and the roofline fraction of the dominant kernel).

Workload (BASELINE.json configs[1], "c1"): elastic, N = 5, fp64, 64^3 Kuhn-split cubes =
1,572,864 tetrahedra, synthetic seeded inputs (synth/).  With --gpus N > 1 (torchrun, one
process per GPU) the mesh is extended to 64 x 64 x 64N cubes and rank r owns the z-slab of
c1's size (weak scaling; the halo of face traces goes over NCCL inside ydg_step).

Timing: W untimed warm-up steps, then K steps bracketed by barrier + synchronize, CUDA
events on the launching stream, max over ranks.  The inputs (6.3 GB of DOFs per GPU) are
larger than L2, so no flush is needed.  Per-kernel device times come from the library's
own CUDA events around each launch (ydg_profile) inside the timed region.

--impl reference times the CPU oracle (oracle/, the test-only reference of this tier) on a
bounded sample of the same workload on the host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

BASELINE = json.load(open(os.path.join(ROOT, "BASELINE.json")))
METRIC = BASELINE["metric"]
UNIT = "element-updates/s"

# Roofline denominators.  MEASURED_PEAKS.json holds only bf16 and HBM, so the
# FP64 / FP32 peaks are this pool's own measurements (tools/peaks.cu -> profiles/peaks_r01.json,
# seconds-long sustained loops, the figure for a kernel timed inside a long step): FP64 DMMA
# (the tensor pipe the fp64 kernels run on; DFMA shares it at the same rate) and FP32 FFMA.
# Fallback: derived from the unit counts and the max clock, 148 SM x 64 FP64 FMA/clk x 2 x
# 1.965 GHz = 37.2 TF/s and twice that for FP32.
_PEAKS_FILE = os.path.join(ROOT, "profiles", "peaks_r01.json")
try:
    _PK = json.load(open(_PEAKS_FILE))
    FP64_PEAK_TFLOPS = float(_PK["fp64_dmma_tflops_sustained"])
    FP32_PEAK_TFLOPS = float(_PK["fp32_fma_tflops_sustained"])
    PEAK_SOURCE = "of measured: profiles/peaks_r01.json (tools/peaks.cu, sustained)"
except (OSError, KeyError, ValueError):
    FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # 37.2
    FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # 74.4
    PEAK_SOURCE = "derived: 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c1")
    ap.add_argument("--impl", default="ydg", choices=["ydg", "reference"])
    ap.add_argument("--replica", type=int, default=0, help="cube count per axis (debug only)")
    ap.add_argument("--e2e-reps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=8, help="cubes per axis of the oracle sample")
    return ap.parse_args()


def workload(args, world):
    cfg = synth.CONFIGS[args.config]
    if args.replica:
        cfg = cfg.replica(args.replica)
    if world > 1:
        cfg = cfg.__class__(**{**cfg.__dict__, "nz": cfg.nz * world, "name": f"{cfg.name}-zslab-x{world}"})
    return cfg


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.file = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.file, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        self.file.flush()
        rows = []
        with open(self.file.name) as fh:
            for line in fh:
                f = [x.strip() for x in line.split(",")]
                if len(f) >= 9:
                    try:
                        rows.append(f)
                    except ValueError:
                        pass
        os.unlink(self.file.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        pw = [float(r[3]) for r in rows if r[3].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        load = [s for s in sm if s > 0]
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(pw) if pw else None, "samples": len(rows), "reasons": reasons}


def dist_setup(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def allmax(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------ oracle (CPU)


def oracle_rate(cfg, cubes, steps, warmup=0):
    """Element-updates/s of the CPU oracle on a periodic cubes^3 sample of cfg (setup untimed)."""
    from oracle import step as ostep
    import threadpoolctl
    sample = cfg.replica(cubes, cubes, cubes)
    xyz, vid = synth.kuhn_mesh(sample.nx, sample.ny, sample.nz, seed=sample.seed)
    mat = synth.material(sample)
    omega = Y = None
    if cfg.P == 27:
        omega, Y = synth.anelastic(sample, mat)
    prob = ostep.setup(cfg.N, xyz, vid, mat, P=cfg.P, omega=omega, Y=Y)
    Q = ostep.to_internal(synth.dofs(sample))
    for _ in range(warmup):
        Q = ostep.step(prob, Q, cfg.dt, 1)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        Q = ostep.step(prob, Q, cfg.dt, 1)
        times.append(time.perf_counter() - t0)
    threads = max([p.get("num_threads", 1) for p in threadpoolctl.threadpool_info()] + [1])
    return sample.n_elements / statistics.mean(times), threads, sample, times


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    cfg = workload(args, world)
    rate, threads, sample, times = oracle_rate(cfg, args.cpu_sample, args.steps, args.warmup)
    desc = (f"oracle (numpy fp64) on {cfg.name} parameters (N={cfg.N}, P={cfg.P}) over a periodic "
            f"{sample.nx}^3-cube sample ({sample.n_elements} elements), one step per timed step")
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "order": cfg.N, "quantities": cfg.P, "sample_elements": sample.n_elements},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": desc},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU path


def load_traffic(cfg_name):
    """dram bytes (read + write) per launch of each kernel from the committed ncu --set full
    capture (profiles/ncu_traffic.json: {workload: {kernel: bytes}})."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return {}
    data = json.load(open(p))
    return data.get(cfg_name, {})


def run_ydg(args):
    import torch
    import paper_1903_11521_b200 as ydg

    rank, world, local = dist_setup(args)
    cfg = workload(args, world)
    t_setup = time.time()
    xyz, vid = synth.kuhn_mesh(cfg.nx, cfg.ny, cfg.nz, seed=cfg.seed, jitter=cfg.jitter)
    mat = synth.material(cfg)
    an = None
    if cfg.P == 27:
        omega, Y = synth.anelastic(cfg, mat)
        an = np.concatenate([omega, Y.ravel()])
    h = ydg.ydg_create(cfg.N, cfg.P, cfg.precision, device=local)
    if world > 1:
        import torch.distributed as dist
        uid = [torch.cuda.nccl.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ydg.ydg_set_comm(h, rank, world, uid[0])
    ydg.ydg_upload_mesh(h, xyz, vid, mat, an)
    del xyz, vid
    first = int(ydg.ydg_query(h, ydg.YDG_Q_FIRST_LOCAL))
    nloc = int(ydg.ydg_query(h, ydg.YDG_Q_N_LOCAL))
    # pinned host DOFs of the owned range (also the e2e input buffer)
    dt_np = np.float64 if cfg.precision == 8 else np.float32
    host = torch.empty((nloc, cfg.P, cfg.B), dtype=torch.float64 if cfg.precision == 8 else torch.float32,
                       pin_memory=True)
    Qh = host.numpy()
    if cfg.precision == 8:
        synth.dofs(cfg, first=first, count=nloc, out=Qh)
    else:
        Qh[...] = synth.dofs(cfg, first=first, count=nloc).astype(dt_np)
    ydg.ydg_upload_dofs(h, first, Qh)
    ydg.ydg_synchronize(h)
    setup_s = time.time() - t_setup
    # a dedicated (non-default) stream: the library enqueues on it and the events below
    # are recorded on it (the legacy default stream would be handle 0 = the library's own)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sptr = stream.cuda_stream
    assert sptr != 0

    # warm-up
    for _ in range(args.warmup):
        ydg.ydg_step(h, cfg.dt, 1, stream=sptr)
    torch.cuda.synchronize()
    barrier(world)

    # timed region
    ydg.ydg_profile(h, True)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        barrier(world)
        e0.record(stream)
        for _ in range(args.steps):
            ydg.ydg_step(h, cfg.dt, 1, stream=sptr)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    ms = e0.elapsed_time(e1)
    clocks = clk.summary()
    t_local = ydg.ydg_query(h, ydg.YDG_Q_PROF_LOCAL_MS)
    t_neigh = ydg.ydg_query(h, ydg.YDG_Q_PROF_NEIGH_MS)
    launches = int(ydg.ydg_query(h, ydg.YDG_Q_PROF_LAUNCHES))
    ydg.ydg_profile(h, False)
    ms_max = allmax(ms, world)
    nz = ydg.ydg_query(h, ydg.YDG_Q_NZ_FLOPS)
    kpath = int(ydg.ydg_query(h, ydg.YDG_Q_KERNEL_PATH))
    fl_local = ydg.ydg_query(h, ydg.YDG_Q_LOCAL_FLOPS)
    fl_neigh = ydg.ydg_query(h, ydg.YDG_Q_NEIGH_FLOPS)
    by_local = ydg.ydg_query(h, ydg.YDG_Q_LOCAL_BYTES)
    by_neigh = ydg.ydg_query(h, ydg.YDG_Q_NEIGH_BYTES)
    per_step_launch = int(ydg.ydg_query(h, ydg.YDG_Q_LAUNCHES_PER_STEP))

    # sampled parity of the benchmarked state is done by tests/; here: NaN guard
    probe = ydg.ydg_download_dofs(h, first, min(nloc, 64))
    finite = bool(np.isfinite(probe).all())

    # e2e: host buffers through the C ABI, copies inside the timed region
    e2e_ms = []
    for _ in range(max(1, args.e2e_reps)):
        barrier(world)
        t0 = time.perf_counter()
        ydg.ydg_upload_dofs(h, first, Qh)
        ydg.ydg_step(h, cfg.dt, cfg.steps)
        ydg.ydg_download_dofs(h, first, nloc, out=Qh)
        e2e_ms.append(1e3 * (time.perf_counter() - t0))
    e2e_best = allmax(min(e2e_ms), world)
    qbytes = nloc * cfg.P * cfg.B * (8 if cfg.precision == 8 else 4)

    if rank != 0:
        ydg.ydg_destroy(h)
        return 0

    ne_total = cfg.n_elements
    value = ne_total * args.steps / (ms_max / 1e3)
    n_launch = args.steps  # launches per kernel kind (single rank: 1 local + 1 neighbour per step)
    if world > 1:
        n_launch_local = max(1, launches - args.steps)
    else:
        n_launch_local = n_launch
    avg_local = t_local / max(1, n_launch_local)
    avg_neigh = t_neigh / max(1, n_launch)
    peak = FP64_PEAK_TFLOPS if cfg.precision == 8 else FP32_PEAK_TFLOPS
    ach_local = fl_local * nloc / (avg_local / 1e3) / 1e12 if world == 1 else fl_local * nloc / (t_local / args.steps / 1e3) / 1e12
    ach_neigh = fl_neigh * nloc / (avg_neigh / 1e3) / 1e12
    # kernel names as ncu lists them, from the path the library reports it runs
    k_loc, k_nb, bound = {0: ("dm_local", "dm_flux", "tensor"), 1: ("ader_local", "ader_neigh", "alu"),
                          2: ("vm_local", "vm_neigh", "tensor"), 3: ("gen_local", "gen_neigh", "alu")}[kpath]
    dominant = k_loc if t_local >= t_neigh else k_nb
    traffic = load_traffic(cfg.name)
    dom_ach = ach_local if dominant == k_loc else ach_neigh
    roofline = {
        "bound": bound, "achieved": round(dom_ach, 3), "peak": round(peak, 2), "unit": "TFLOP/s",
        "frac": round(dom_ach / peak, 4), "traffic": traffic.get(dominant),
        "kernel": dominant, "peak_source": PEAK_SOURCE,
        "algorithmic_flops_per_element": fl_local if dominant == k_loc else fl_neigh,
        "elements_per_launch": nloc,
    }
    kernels = {
        k_loc: {"ms_per_launch": round(avg_local, 4), "tflops": round(ach_local, 3),
                "frac_peak": round(ach_local / peak, 4),
                "alg_hbm_gbs": round(by_local * nloc / (avg_local / 1e3) / 1e9, 1),
                "nz_flops_per_element": fl_local, "alg_bytes_per_element": by_local},
        k_nb: {"ms_per_launch": round(avg_neigh, 4), "tflops": round(ach_neigh, 3),
               "frac_peak": round(ach_neigh / peak, 4),
               "alg_hbm_gbs": round(by_neigh * nloc / (avg_neigh / 1e3) / 1e9, 1),
               "nz_flops_per_element": fl_neigh, "alg_bytes_per_element": by_neigh},
    }
    step_roof = peak * 1e12 / nz  # element-updates/s if the whole step ran at the FP64 peak
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        rate, threads, sample, times = oracle_rate(cfg, args.cpu_sample, 2, 0)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "oracle",
               "sample": f"oracle (numpy fp64) on {cfg.name} parameters over a periodic {sample.nx}^3-cube "
                         f"sample ({sample.n_elements} elements), mean of 2 steps, setup untimed"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64" if cfg.precision == 8 else "f32",
        "data": "synthetic",
        "config": {"workload": cfg.name, "model": "ADER-DG elastic tetrahedra" if cfg.P == 9 else "ADER-DG viscoelastic",
                   "order": cfg.N, "quantities": cfg.P, "elements": ne_total, "elements_per_gpu": nloc,
                   "mesh": f"{cfg.nx}x{cfg.ny}x{cfg.nz} Kuhn cubes, periodic", "dt": cfg.dt,
                   "parallelism": f"zslab{world}" if world > 1 else "single",
                   "l2": "inputs larger than L2 (DOFs %.1f GB/GPU), no flush" % (qbytes / 1e9)},
        "nz_gflops": value * nz / 1e9, "nz_flops_per_element": nz,
        "dof_updates_per_s": value * cfg.B * cfg.P,
        "step_roofline_frac": value / world / step_roof,
        "roofline": roofline, "kernels": kernels,
        "cpu_baseline": cpu,
        "e2e": {"value": ne_total * cfg.steps / (e2e_best / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": qbytes * world / cfg.steps, "d2h_bytes_per_step": qbytes * world / cfg.steps,
                "steps_per_call": cfg.steps,
                "call": "ydg_upload_dofs(pinned host) + ydg_step(dt, %d) + ydg_download_dofs(pinned host)" % cfg.steps},
        "gpu_launches": args.steps * per_step_launch,
        "clocks": clocks, "finite": finite, "setup_s": round(setup_s, 1),
    }
    print(json.dumps(line), flush=True)
    ydg.ydg_destroy(h)
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ydg(args)


if __name__ == "__main__":
    sys.exit(main())
