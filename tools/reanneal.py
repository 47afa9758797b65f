"""Re-anneal the cached DMMA row groupings with the incremental-cost annealer (tools/anneal.c).

    python tools/reanneal.py N [--moves 6000000] [--restarts 24] [--only ck0,vol] [--visco]

Every product of gen/tiling.products(N) is searched from `restarts` random starts in
parallel; a result replaces the cached grouping only if gen/tiling's own cost function
(the definition) confirms a lower tile count.
"""
import argparse
import os
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1903_11521_b200.gen import tiling  # noqa: E402


def solve(name, pr, moves, restarts, exe, workers):
    mats, classes = pr[0], pr[1]
    part_of = pr[2] if len(pr) > 2 else [0] * len(mats)
    nout, nin = mats[0].shape
    cls = [-1] * nin
    for ci, cl in enumerate(classes):
        for j in cl:
            cls[j] = ci
    assert min(cls) >= 0
    with tempfile.NamedTemporaryFile("w", suffix=".txt", delete=False) as fh:
        fh.write(f"{len(mats)} {nout} {nin} {max(part_of) + 1}\n")
        fh.write(" ".join(map(str, part_of)) + "\n" + " ".join(map(str, cls)) + "\n")
        for m in mats:
            for row in np.asarray(m, dtype=int):
                fh.write(" ".join(map(str, row)) + "\n")
        path = fh.name

    def run(seed):
        out = subprocess.run([exe, path, str(moves), str(seed)], capture_output=True, text=True, check=True).stdout.split("\n")
        return int(out[0]), [int(x) for x in out[1].split()], [[int(x) for x in l.split()] for l in out[2:] if l.strip()]

    with ThreadPoolExecutor(workers) as ex:
        res = list(ex.map(run, range(1, restarts + 1)))
    os.unlink(path)
    cost, og_of, ig_of = min(res, key=lambda r: r[0])
    og = [sorted(r for r in range(nout) if og_of[r] == g) for g in range(max(og_of) + 1)]
    igs = [[sorted(j for j in range(nin) if ig[j] == g) for g in range(max(ig) + 1)] for ig in ig_of]
    prob = tiling._Problem(mats, nin, part_of)
    check = prob.cost(og, igs)
    assert check == cost, (name, check, cost)
    assert all(len(g) <= 8 for g in og) and all(len(g) <= 4 for ig in igs for g in ig)
    return {"tiles": cost, "out": og, "in": igs}, sorted(r[0] for r in res)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("N", type=int)
    ap.add_argument("--moves", type=int, default=6_000_000)
    ap.add_argument("--restarts", type=int, default=24)
    ap.add_argument("--only", default="")
    ap.add_argument("--workers", type=int, default=os.cpu_count())
    a = ap.parse_args()
    exe = "/tmp/ydg_anneal"
    subprocess.run(["gcc", "-O2", "-o", exe, os.path.join(ROOT, "tools", "anneal.c"), "-lm"], check=True)
    cur = tiling.tiling(a.N)
    for name, pr in tiling.products(a.N).items():
        if a.only and name not in a.only.split(","):
            continue
        new, costs = solve(name, pr, a.moves, a.restarts, exe, a.workers)
        old = cur[name]["tiles"]
        print(f"N={a.N} {name}: cached {old}, annealed {new['tiles']} (restarts: {costs[:6]}...)", flush=True)
        if new["tiles"] < old:
            cur[name] = new
            tiling._store(a.N, cur)
