"""Hardware flops per element-update measured from an ncu source capture (the paper's
"hardware flops", counted from the executed SASS instead of the generator):
DMMA m8n8k4 = 512 flops per warp instruction; DFMA / FFMA 2, FFMA2 4, DMUL / DADD / FMUL /
FADD 1 per predicated-on thread.

    ncu -i REPORT --page source --csv --print-source sass > src.csv
    python tools/hw_flops.py src.csv ELEMENTS_PER_LAUNCH
"""
import csv
import json
import re
import sys

PER_THREAD = {"DFMA": 2, "FFMA": 2, "FFMA2": 4, "DMUL": 1, "DADD": 1, "FMUL": 1, "FADD": 1}


def hw_flops(path, elements):
    rows = list(csv.reader(open(path)))
    kern = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
    out = {}
    for w, k in enumerate(kern):
        hdr = rows[k + 1]
        ci = {h: i for i, h in enumerate(hdr)}
        end = kern[w + 1] if w + 1 < len(kern) else len(rows)
        fl = {}
        for r in rows[k + 2:end]:
            src = re.sub(r"^@!?U?P\w+\s+", "", r[1].strip())
            op = src.split()[0].split(".")[0] if src else ""
            if op == "DMMA":
                fl[op] = fl.get(op, 0) + 512 * int(r[ci["Instructions Executed"]] or 0)
            elif op in PER_THREAD:
                n = int(r[ci["Predicated-On Thread Instructions Executed"]] or 0)
                fl[op] = fl.get(op, 0) + PER_THREAD[op] * n
        short = re.search(r"(\w+)<", rows[k][1]).group(1)
        out.setdefault(short, {"hw_flops_per_element": sum(fl.values()) / elements,
                               "by_op_per_element": {a: b / elements for a, b in fl.items()}})
    return out


if __name__ == "__main__":
    print(json.dumps(hw_flops(sys.argv[1], float(sys.argv[2])), indent=1))
