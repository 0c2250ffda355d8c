"""Register / stack / spill report for generated kernels (compiles the
generated source with nvcc -Xptxas -v for sm_100a; no GPU needed).

    python tools/kstat.py c2 [--dtypes f32,f64]
"""
import argparse
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2501_13986_b200 as cgf  # noqa: E402
from oracle.oracle import CONFIGS, config_json  # noqa: E402

KERNELS = [("tp_fwd", 0, 0), ("tp_bwd", 1, 0), ("tp_dbwd", 2, 0), ("convo_fwd", 0, 1), ("convo_dbwdz", 3, 1),
           ("convi_bwd", 1, 2), ("convi_dbwdx", 4, 2)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("problem")
    ap.add_argument("--dtypes", default="f32,f64")
    ap.add_argument("--kernels", default=",".join(k[0] for k in KERNELS))
    ap.add_argument("--keep", default="")
    a = ap.parse_args()
    if a.problem in CONFIGS:
        js = config_json(a.problem)
    else:
        from problems import random_problem
        js = random_problem(int(a.problem))
    plan = cgf.TpPlan(js)
    want = set(a.kernels.split(","))
    for name, comp, loop in KERNELS:
        if name not in want:
            continue
        for dt in a.dtypes.split(","):
            src = cgf._kernel_source(plan, comp, loop, 0 if dt == "f32" else 1)
            with tempfile.TemporaryDirectory() as d:
                f = os.path.join(d, "k.cu")
                open(f, "w").write(src)
                if a.keep:
                    open(f"{a.keep}_{name}_{dt}.cu", "w").write(src)
                r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17", "-cubin",
                                    "-Xptxas", "-v", "-o", os.path.join(d, "k.cubin"), f],
                                   capture_output=True, text=True)
                log = r.stdout + r.stderr
                regs = re.search(r"Used (\d+) registers", log)
                stack = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", log)
                smem = re.search(r"threads (\d+) smem (\d+)", "")
                print(f"{a.problem:6s} {name:12s} {dt}: regs {regs.group(1) if regs else '?':>4s} "
                      f"stack {stack.group(1) if stack else '?':>5s} spill st/ld "
                      f"{stack.group(2) if stack else '?'}/{stack.group(3) if stack else '?'}  "
                      f"src {len(src)//1024} KB" + ("" if r.returncode == 0 else "  COMPILE FAILED"), flush=True)


if __name__ == "__main__":
    main()
