"""Small runs of every kernel family through the C ABI, for compute-sanitizer (one tool per
gpurun call: memcheck, racecheck, synccheck, initcheck).  Each case steps a small mesh and
checks the result against the oracle, so a tool-induced change of results also shows.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from tests.helpers import check_parity, make_inputs, rel_err, run_gpu, run_oracle  # noqa: E402

CASES = [
    ("c0 fp64 dm_local/dm_flux (N=2)", synth.CONFIGS["c0"].with_(vperm=True), {}),
    ("c1 replica fp64 dm_local/dm_flux (N=5)", synth.CONFIGS["c1"].replica(3, steps=2).with_(vperm=True), {}),
    ("c2 replica fp32 ader_local/ader_neigh (N=6)", synth.CONFIGS["c2"].replica(3, steps=1).with_(vperm=True), {}),
    ("c3 replica visco vm_local/vm_neigh (N=4)", synth.CONFIGS["c3"].replica(3, steps=1).with_(vperm=True), {}),
    ("generic gen_local/gen_neigh (N=6 fp64)", synth.CONFIGS["c1"].with_(N=6, nx=3, ny=3, nz=3, steps=1), {}),
]

if __name__ == "__main__":
    for label, cfg, env in CASES:
        os.environ.update(env)
        xyz, vid, mat, Q, an = make_inputs(cfg)
        got, _ = run_gpu(cfg, xyz, vid, mat, Q, an)
        ref = run_oracle(cfg, xyz, vid, mat, Q, an)
        check_parity(rel_err(got, ref), cfg.precision, label)
    print("sanitize cases done")
