#!/usr/bin/env python
"""Benchmark of the B200 ADER-DG element update (arXiv:1903.11521 Sec. 5.1).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1] [--impl ydg|reference]

One *step* = one global ADER-DG time step of every element of the workload (the whole hot
path: CK recursion, time integral, volume, local and neighbour flux = BASELINE.json
north_star): two kernel launches (local part, flux).  The K timed steps are one
``ydg_step(dt, K)`` call, as a user advancing a simulation makes it.  Metric: element-
updates/s (plus nonzero GFLOP/s and the roofline fraction of the dominant kernel).

Workload (BASELINE.json configs[1], "c1"): elastic, N = 5, fp64, 64^3 Kuhn-split cubes =
1,572,864 tetrahedra, synthetic seeded inputs (synth/).  With --gpus N > 1 (one process per
GPU; launched under torchrun by the driver, or re-executed under torchrun by this script
when WORLD_SIZE is unset) the mesh is extended to 64 x 64 x 64N cubes and rank r owns the
z-slab of c1's size (weak scaling; the halo of shared-face traces goes over NCCL inside
ydg_step).  --config c4 (BASELINE configs[4]) is strong scaling: the fixed 128^3-cube mesh
(12,582,912 tetrahedra) split into N z-slabs of 128/N cube layers.

Timing: W untimed warm-up steps (one call), then K steps bracketed by barrier + synchronize, CUDA
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
    ap.add_argument("--sims", type=int, default=1,
                    help="fused simulations S (NEXT-1, P:1306-1308): element-simulations = elements x S")
    ap.add_argument("--lts", action="store_true",
                    help="NEXT-2: two-cluster local time stepping on the config's mesh with the two-layer "
                         "material (upper half vp in [1500, 2500] advances by 2 dt); reports GTS-equivalent "
                         "element-updates/s and the speed-up over global time stepping on the same mesh")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="time ydg_step_graph (one CUDA graph per step); auto: on below 100k elements "
                         "(c0: launch-latency bound), 1 GPU only")
    return ap.parse_args()


STRONG = ("c4",)  # configs with a fixed global mesh (strong scaling over z-slabs)


def workload(args, world):
    cfg = synth.CONFIGS[args.config]
    if args.replica:
        cfg = cfg.replica(args.replica)
    if world > 1 and args.config not in STRONG:
        cfg = cfg.__class__(**{**cfg.__dict__, "nz": cfg.nz * world, "name": f"{cfg.name}-zslab-x{world}"})
    return cfg


def relaunch_under_torchrun(args):
    """--gpus N > 1 without a torchrun environment: run this script as N ranks (one per GPU)
    under torch.distributed.run on 127.0.0.1 and pass its exit code through."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


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


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def oracle_rate(cfg, cubes, steps, warmup=0, threads=None):
    """Element-updates/s of the CPU oracle on a periodic cubes^3 sample of cfg (setup untimed),
    BLAS/OpenMP pools limited to `threads` (None: every host core)."""
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
    nthreads = threads or os.cpu_count() or 1
    with threadpoolctl.threadpool_limits(nthreads):
        for _ in range(warmup):
            Q = ostep.step(prob, Q, cfg.dt, 1)
        times = []
        for _ in range(steps):
            t0 = time.perf_counter()
            Q = ostep.step(prob, Q, cfg.dt, 1)
            times.append(time.perf_counter() - t0)
        used = max([p.get("num_threads", 1) for p in threadpoolctl.threadpool_info()] + [1])
    return sample.n_elements / statistics.mean(times), used, sample, times


def cpu_baseline(cfg, cubes, steps=5):
    """The oracle on all host cores (cubes^3 sample) and on one core (a 4^3 sample): min and
    median of `steps` timed steps after one warm-up step each."""
    _, used, sample, times = oracle_rate(cfg, cubes, steps, 1)
    _, _, sample1, times1 = oracle_rate(cfg, 4, steps, 1, threads=1)
    rate = sample.n_elements / statistics.median(times)
    return {
        "value": rate, "unit": UNIT, "cores": used, "kind": "oracle",
        "sample": (f"oracle (numpy fp64) on {cfg.name} parameters (N={cfg.N}, P={cfg.P}) over a periodic "
                   f"{sample.nx}^3-cube sample ({sample.n_elements} elements); value = median of {steps} "
                   f"steps after 1 warm-up, setup untimed"),
        "all_cores": {"median": rate, "best": sample.n_elements / min(times), "threads": used,
                      "elements": sample.n_elements, "steps": steps},
        "single_core": {"median": sample1.n_elements / statistics.median(times1),
                        "best": sample1.n_elements / min(times1), "elements": sample1.n_elements, "steps": steps},
        "host_cores": os.cpu_count(), "cpu_model": cpu_model(),
    }


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    cfg = workload(args, world)
    rate, threads, sample, times = oracle_rate(cfg, args.cpu_sample, args.steps, args.warmup)
    desc = (f"oracle (numpy fp64) on {cfg.name} parameters (N={cfg.N}, P={cfg.P}) over a periodic "
            f"{sample.nx}^3-cube sample ({sample.n_elements} elements), one step per timed step, "
            f"{threads} threads on {os.cpu_count()} host cores ({cpu_model()})")
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "order": cfg.N, "quantities": cfg.P, "sample_elements": sample.n_elements},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": desc,
                         "best": sample.n_elements / min(times), "median": sample.n_elements / statistics.median(times)},
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


def load_hw_flops(cfg_name):
    """Hardware flops per element of each kernel (DMMA 512 per warp instruction, DFMA 2,
    DMUL / DADD 1 per thread, from the executed SASS of a committed ncu source capture:
    profiles/hw_flops.json {workload: {kernel: flops}}, tools/hw_flops.py) -- the paper's
    "hardware flops" beside the nonzero flops."""
    p = os.path.join(ROOT, "profiles", "hw_flops.json")
    if not os.path.exists(p):
        return {}
    return json.load(open(p)).get(cfg_name, {})


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
    if args.sims > 1:
        ydg.ydg_set_simulations(h, args.sims)
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

    qbytes = nloc * cfg.P * cfg.B * (8 if cfg.precision == 8 else 4)
    # inputs smaller than L2 (126 MB): a 512 MB buffer is rewritten between timed steps
    flush = torch.zeros(64 << 20, dtype=torch.float64, device="cuda") if 4 * qbytes < 126e6 else None
    use_graph = world == 1 and (args.graph == "on" or (args.graph == "auto" and cfg.n_elements < 100000))
    step_fn = ydg.ydg_step_graph if use_graph else ydg.ydg_step

    # warm-up (one call of W steps on the large workloads: the same launch sequence as the
    # timed call, fused kernels included)
    if flush is None:
        step_fn(h, cfg.dt, args.warmup, stream=sptr)
    else:
        for _ in range(args.warmup):
            step_fn(h, cfg.dt, 1, stream=sptr)
    torch.cuda.synchronize()
    # the timed steps start from the config's initial state again (the configs' dt exceeds
    # the CFL bound, DESIGN R13/R27: W + K steps of growth would overflow fp32 sooner)
    ydg.ydg_upload_dofs(h, first, Qh)
    ydg.ydg_synchronize(h)
    barrier(world)

    # timed region (per-kernel events inside it, except on the graph path: there the same
    # steps are replayed once more with the events, after the timed region)
    if not use_graph:
        ydg.ydg_profile(h, True)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        barrier(world)
        if flush is None:  # K steps in one call (what a user advancing a simulation does)
            e0.record(stream)
            step_fn(h, cfg.dt, args.steps, stream=sptr)
            e1.record(stream)
        else:  # L2-resident workload: flush L2 between steps, time each step on its own
            evs = []
            for _ in range(args.steps):
                flush.add_(1)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                step_fn(h, cfg.dt, 1, stream=sptr)
                b.record(stream)
                evs.append((a, b))
        torch.cuda.synchronize()
        barrier(world)
    ms = e0.elapsed_time(e1) if flush is None else sum(a.elapsed_time(b) for a, b in evs)
    clocks = clk.summary()
    if use_graph:
        ydg.ydg_profile(h, True)
        for _ in range(args.steps):
            ydg.ydg_step(h, cfg.dt, 1, stream=sptr)
        torch.cuda.synchronize()
    t_local = ydg.ydg_query(h, ydg.YDG_Q_PROF_LOCAL_MS)
    t_neigh = ydg.ydg_query(h, ydg.YDG_Q_PROF_NEIGH_MS)
    t_fused = ydg.ydg_query(h, ydg.YDG_Q_PROF_FUSED_MS)
    # fused step kernel (one rank, fp64, K >= 2 steps in one call): local(0), K - 1 fused, flux(K - 1)
    fused = world == 1 and flush is None and args.steps >= 2 and ydg.ydg_query(h, ydg.YDG_Q_FUSED) == 1.0
    launches = int(ydg.ydg_query(h, ydg.YDG_Q_PROF_LAUNCHES))
    ydg.ydg_profile(h, False)
    ms_max = allmax(ms, world)
    nz = ydg.ydg_query(h, ydg.YDG_Q_NZ_FLOPS)
    kpath = int(ydg.ydg_query(h, ydg.YDG_Q_KERNEL_PATH))
    fl_local = ydg.ydg_query(h, ydg.YDG_Q_LOCAL_FLOPS)
    fl_neigh = ydg.ydg_query(h, ydg.YDG_Q_NEIGH_FLOPS)
    fl_neigh_exec = ydg.ydg_query(h, ydg.YDG_Q_NEIGH_FLOPS_EXEC)
    by_local = ydg.ydg_query(h, ydg.YDG_Q_LOCAL_BYTES)
    by_neigh = ydg.ydg_query(h, ydg.YDG_Q_NEIGH_BYTES)
    per_step_launch = int(ydg.ydg_query(h, ydg.YDG_Q_LAUNCHES_PER_STEP))

    # sampled parity of the benchmarked state is done by tests/; here: the max|Q| diagnostic
    # over every owned DOF (a reduction kernel, after the timed region), NaN if any is not finite
    max_abs_q = ydg.ydg_query(h, ydg.YDG_Q_MAX_ABS_Q)
    finite = bool(np.isfinite(max_abs_q))

    # e2e: host buffers through the C ABI, copies inside the timed region
    e2e_ms = []
    for _ in range(max(1, args.e2e_reps)):
        barrier(world)
        t0 = time.perf_counter()
        ydg.ydg_upload_dofs(h, first, Qh)
        step_fn(h, cfg.dt, cfg.steps)
        ydg.ydg_download_dofs(h, first, nloc, out=Qh)
        e2e_ms.append(1e3 * (time.perf_counter() - t0))
    e2e_best = allmax(min(e2e_ms), world)

    if rank != 0:
        ydg.ydg_destroy(h)
        return 0

    ne_total = cfg.n_elements * args.sims  # element-simulations with fused simulations
    value = ne_total * args.steps / (ms_max / 1e3)
    n_launch = args.steps  # launches per kernel kind (single rank: 1 local + 1 neighbour per step)
    if fused:
        n_launch = n_launch_local = 1
    elif world > 1:
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
    dom_fl = fl_local if dominant == k_loc else fl_neigh
    if fused:  # the fused kernel carries K - 1 of the K steps: it is the dominant kernel
        avg_fused = t_fused / (args.steps - 1)
        dominant, dom_fl = "dm_fused", fl_local + fl_neigh
        dom_ach = dom_fl * nloc / (avg_fused / 1e3) / 1e12
    roofline = {
        "bound": bound, "achieved": round(dom_ach, 3), "peak": round(peak, 2), "unit": "TFLOP/s",
        "frac": round(dom_ach / peak, 4), "traffic": traffic.get(dominant),
        "kernel": dominant, "peak_source": PEAK_SOURCE,
        "algorithmic_flops_per_element": dom_fl,
        "elements_per_launch": nloc,
    }
    kernels = {
        k_loc: {"ms_per_launch": round(avg_local, 4), "tflops": round(ach_local, 3),
                "frac_peak": round(ach_local / peak, 4),
                "alg_hbm_gbs": round(by_local * nloc / (avg_local / 1e3) / 1e9, 1),
                "nz_flops_per_element": fl_local, "alg_bytes_per_element": by_local},
        k_nb: {"ms_per_launch": round(avg_neigh, 4), "tflops": round(ach_neigh, 3),
               "frac_peak": round(ach_neigh / peak, 4),
               "executed_nz_flops_per_element": fl_neigh_exec,
               "frac_peak_executed": round(ach_neigh * fl_neigh_exec / fl_neigh / peak, 4) if fl_neigh else None,
               "alg_hbm_gbs": round(by_neigh * nloc / (avg_neigh / 1e3) / 1e9, 1),
               "nz_flops_per_element": fl_neigh, "alg_bytes_per_element": by_neigh},
    }
    if fused:
        by_fused = ydg.ydg_query(h, ydg.YDG_Q_FUSED_BYTES)
        kernels["dm_fused"] = {
            "ms_per_launch": round(avg_fused, 4), "launches": args.steps - 1, "tflops": round(dom_ach, 3),
            "frac_peak": round(dom_ach / peak, 4),
            "frac_peak_executed": round(dom_ach * (fl_local + fl_neigh_exec) / dom_fl / peak, 4),
            "alg_hbm_gbs": round(by_fused * nloc / (avg_fused / 1e3) / 1e9, 1),
            "nz_flops_per_element": dom_fl, "executed_nz_flops_per_element": fl_local + fl_neigh_exec,
            "alg_bytes_per_element": by_fused,
            "what": "flux of step n-1 + local part of step n per tile (one launch per step after the first)"}
        kernels[k_loc]["launches"] = kernels[k_nb]["launches"] = 1
    hw = load_hw_flops(cfg.name) if args.sims == 1 else {}
    for kname, avg in ((k_loc, avg_local), (k_nb, avg_neigh)):
        f = hw.get(kname)
        if f:
            kernels[kname]["hw_flops_per_element"] = f
            kernels[kname]["hw_tflops"] = round(f * nloc / (avg / 1e3) / 1e12, 3)
            kernels[kname]["hw_frac_peak"] = round(f * nloc / (avg / 1e3) / 1e12 / peak, 4)
    hw_step = sum(hw.get(k, 0.0) for k in (k_loc, k_nb)) if all(hw.get(k) for k in (k_loc, k_nb)) else None
    step_roof = peak * 1e12 / nz  # element-updates/s if the whole step ran at the FP64 peak
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, args.cpu_sample)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.config in STRONG else "weak", "vs_baseline": None,
        "dtype": "f64" if cfg.precision == 8 else "f32",
        "data": "synthetic",
        "config": {"workload": cfg.name + (f"-S{args.sims}" if args.sims > 1 else ""), "simulations": args.sims,
                   "model": "ADER-DG elastic tetrahedra" if cfg.P == 9 else "ADER-DG viscoelastic",
                   "order": cfg.N, "quantities": cfg.P, "elements": ne_total, "elements_per_gpu": nloc,
                   "mesh": f"{cfg.nx}x{cfg.ny}x{cfg.nz} Kuhn cubes, periodic", "dt": cfg.dt,
                   "parallelism": f"zslab{world}" if world > 1 else "single",
                   "device_bytes_per_gpu": int(ydg.ydg_query(h, ydg.YDG_Q_DEVICE_BYTES)),
                   "l2": ("inputs larger than L2 (DOFs %.1f GB/GPU), no flush" % (qbytes / 1e9)) if flush is None
                         else "L2 flushed (512 MB rewrite) before every timed step; steps timed one by one"},
        "nz_gflops": value * nz / 1e9, "nz_flops_per_element": nz,
        "hw_gflops": value * hw_step / 1e9 if hw_step else None, "hw_flops_per_element": hw_step,
        "dof_updates_per_s": value * cfg.B * cfg.P,
        "step_roofline_frac": value / world / step_roof,
        "roofline": roofline, "kernels": kernels,
        "cpu_baseline": cpu,
        "e2e": {"value": ne_total * cfg.steps / (e2e_best / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": qbytes * world / cfg.steps, "d2h_bytes_per_step": qbytes * world / cfg.steps,
                "steps_per_call": cfg.steps,
                "call": "ydg_upload_dofs(pinned host) + %s(dt, %d) + ydg_download_dofs(pinned host)"
                        % ("ydg_step_graph" if use_graph else "ydg_step", cfg.steps)},
        "gpu_launches": (args.steps + 1 if fused else args.steps * per_step_launch), "cuda_graph": use_graph,
        "fused_step_kernel": fused,
        "clocks": clocks, "finite": finite, "max_abs_q": max_abs_q, "setup_s": round(setup_s, 1),
    }
    print(json.dumps(line), flush=True)
    ydg.ydg_destroy(h)
    return 0


def run_lina(args):
    """LinA workload (NEXT-3): ADER-DG-SEM acoustics, order 8, 64^3 cuboids."""
    import torch
    import paper_1903_11521_b200 as ydg
    rank, world, local = dist_setup(args)
    if world > 1:
        if rank == 0:
            print(json.dumps({"error": "the LinA workload runs on one GPU"}), flush=True)
        return 0
    cfg = synth.LINA_CONFIGS[args.config]
    if args.replica:
        cfg = cfg.with_(nx=args.replica, ny=args.replica, nz=args.replica)
    mat = synth.lina_material(cfg)
    h = ydg.lina_create(cfg.N, 8, local)
    ydg.lina_upload_grid(h, cfg.nx, cfg.ny, cfg.nz, np.array(cfg.h), mat)
    n = cfg.N + 1
    E = cfg.n_elements
    host = torch.empty((E, 4, n, n, n), dtype=torch.float64, pin_memory=True)
    Qh = host.numpy()
    Qh[...] = synth.lina_dofs(cfg)
    ydg.lina_upload_dofs(h, 0, Qh)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sptr = stream.cuda_stream
    for _ in range(args.warmup):
        ydg.lina_step(h, cfg.dt, 1, stream=sptr)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            ydg.lina_step(h, cfg.dt, 1, stream=sptr)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    clocks = clk.summary()
    flops = ydg.lina_query(h, ydg.LINA_Q_NZ_FLOPS)
    abytes = ydg.lina_query(h, ydg.LINA_Q_ALG_BYTES)
    probe = ydg.lina_download_dofs(h, 0, min(E, 16))
    e2e = []
    for _ in range(max(1, args.e2e_reps)):
        t0 = time.perf_counter()
        ydg.lina_upload_dofs(h, 0, Qh)
        ydg.lina_step(h, cfg.dt, cfg.steps)
        Qh[...] = ydg.lina_download_dofs(h, 0, E)
        e2e.append(1e3 * (time.perf_counter() - t0))
    value = E * args.steps / (ms / 1e3)
    ach = value * flops / 1e12
    qbytes = E * 4 * n ** 3 * 8
    cpu = None
    if not args.no_cpu_baseline:
        from oracle import lina as olina
        small = cfg.with_(nx=4, ny=4, nz=4)
        g = olina.setup(small.N, small.nx, small.ny, small.nz, small.h, synth.lina_material(small))
        Qs = np.ascontiguousarray(synth.lina_dofs(small).transpose(0, 2, 3, 4, 1))
        olina.step(g, Qs, small.dt, 1)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            olina.step(g, Qs, small.dt, 1)
            ts.append(time.perf_counter() - t0)
        cpu = {"value": small.n_elements / statistics.median(ts), "unit": UNIT, "cores": os.cpu_count(),
               "kind": "oracle", "sample": f"oracle/lina.py on a 4^3-element grid at N={small.N}, median of 3 steps"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "model": "LinA ADER-DG-SEM acoustics (NEXT-3)", "order": cfg.N + 1,
                   "elements": E, "grid": f"{cfg.nx}x{cfg.ny}x{cfg.nz} periodic cuboids", "dt": cfg.dt,
                   "l2": "inputs larger than L2 (DOFs %.1f GB), no flush" % (qbytes / 1e9)},
        "nz_flops_per_element": flops, "nz_gflops": value * flops / 1e9,
        "roofline": {"bound": "alu", "achieved": round(ach, 3), "peak": round(FP64_PEAK_TFLOPS, 2),
                     "unit": "TFLOP/s", "frac": round(ach / FP64_PEAK_TFLOPS, 4), "traffic": None,
                     "kernel": "lina_local+lina_flux (whole step)", "peak_source": PEAK_SOURCE,
                     "alg_hbm_gbs": round(value * abytes / 1e9, 1), "alg_bytes_per_element": abytes},
        "cpu_baseline": cpu,
        "e2e": {"value": E * cfg.steps / (min(e2e) / 1e3), "unit": UNIT, "h2d_bytes_per_step": qbytes / cfg.steps,
                "d2h_bytes_per_step": qbytes / cfg.steps, "steps_per_call": cfg.steps},
        "gpu_launches": 2 * args.steps, "clocks": clocks, "finite": bool(np.isfinite(probe).all()),
    }
    print(json.dumps(line), flush=True)
    ydg.lina_destroy(h)
    return 0


def run_lts(args):
    """LTS (NEXT-2, reading R26) vs GTS on one handle: c1's mesh and order with the two-layer
    material; a cycle advances every element by 2 dt (= two GTS steps of dt)."""
    import torch
    import paper_1903_11521_b200 as ydg
    rank, world, local = dist_setup(args)
    if world > 1:
        if rank == 0:
            print(json.dumps({"error": "LTS runs on one GPU"}), flush=True)
        return 0
    cfg = synth.CONFIGS[args.config].with_(material="two_layer", name=args.config + "-lts")
    if args.replica:
        cfg = cfg.replica(args.replica)
    xyz, vid = synth.mesh(cfg)
    mat = synth.material(cfg)
    cl = (xyz[:, :, 2].mean(1) >= cfg.nz / 2).astype(np.int8)  # upper half: slow layer, 2 dt
    vp_c, vp_f = mat[cl == 1, 1].max(), mat[cl == 0, 1].max()
    assert 2 * vp_c <= vp_f, "coarse cluster must be CFL-admissible at 2 dt"
    h = ydg.ydg_create(cfg.N, cfg.P, cfg.precision, device=local)
    ydg.ydg_set_clusters(h, cl)
    ydg.ydg_upload_mesh(h, xyz, vid, mat)
    E = cfg.n_elements
    del xyz, vid
    ydg.ydg_upload_dofs(h, 0, synth.dofs(cfg))
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sptr = stream.cuda_stream
    dt = 0.5 * cfg.dt  # fine step: the GTS step of the fast layer
    res = {}
    for mode in ("lts", "gts"):
        for _ in range(args.warmup):
            if mode == "lts":
                ydg.ydg_step_lts(h, dt, 1, stream=sptr)
            else:
                ydg.ydg_step(h, dt, 2, stream=sptr)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with Clocks(local) as clk:
            e0.record(stream)
            for _ in range(args.steps):  # one step = 2 dt of simulated time
                if mode == "lts":
                    ydg.ydg_step_lts(h, dt, 1, stream=sptr)
                else:
                    ydg.ydg_step(h, dt, 2, stream=sptr)
            e1.record(stream)
            torch.cuda.synchronize()
        res[mode] = (e0.elapsed_time(e1), clk.summary())
    ms, clocks = res["lts"]
    value = 2 * E * args.steps / (ms / 1e3)
    gts_value = 2 * E * args.steps / (res["gts"][0] / 1e3)
    nz = ydg.ydg_query(h, ydg.YDG_Q_NZ_FLOPS)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT + " (GTS-equivalent: element x dt advanced)",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "order": cfg.N, "elements": E, "coarse_elements": int(cl.sum()),
                   "dt_fine": dt, "step": "one LTS cycle = 2 dt of simulated time",
                   "material": "two-layer: upper half vp in [1500, 2500] (cluster 1, 2 dt), lower [4000, 6000]",
                   "l2": "inputs larger than L2, no flush"},
        "gts": {"value": gts_value, "ms_per_2dt": res["gts"][0] / args.steps},
        "lts_speedup_vs_gts": value / gts_value,
        "nz_gflops_equivalent": value * nz / 1e9, "clocks": clocks,
        "gpu_launches": 10 * args.steps,
    }
    print(json.dumps(line), flush=True)
    ydg.ydg_destroy(h)
    return 0


def main():
    args = parse()
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is None and args.gpus > 1:
        return relaunch_under_torchrun(args)
    if world_env is not None and int(world_env) != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world_env}"}), flush=True)
        return 2
    if args.lts:
        return run_lts(args)
    if args.config.startswith("lina"):
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "the reference arm times the c-configs"}))
            return 0
        return run_lina(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ydg(args)


if __name__ == "__main__":
    sys.exit(main())
