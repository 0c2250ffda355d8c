"""SASS opcode counts of the generated kernels (cuobjdump -sass of the NVRTC
cubins): the evidence that the hot kernels use TMA / bulk copies
(UTMALDG / UBLKCP), cp.async (LDGSTS), tcgen05 MMAs (UTC*MMA) and TMEM
(LDTM / STTM), and how big each kernel's code is (instruction-cache pressure).

    python tools/sass_stats.py > profiles/r02_sass_opcodes.json
"""
import collections
import glob
import json
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

KEY = ("FFMA", "FFMA2", "FMUL", "FMUL2", "FADD", "DFMA", "DMUL", "DADD", "LDS", "STS", "LDG", "STG", "LDGSTS", "UBLKCP", "UTMALDG",
       "UTMASTG", "UTCHMMA", "UTCQMMA", "UTCMMA", "LDTM", "STTM", "SYNCS", "RED", "ATOM", "BRA", "SHFL")


def main():
    import paper_2501_13986_b200 as cgf
    from paper_2501_13986_b200.configs import config_json
    # per config, every kernel the bench and the BASELINE configs launch: (comp, loop, dtype)
    jobs = {"c1": [(c, 0, d) for c in (0, 1, 2) for d in (0, 1)] + [(0, 1, 0), (1, 2, 0), (3, 1, 0), (4, 2, 0)],
            "c2": [(c, 0, d) for c in (0, 1, 2) for d in (0, 1)] + [(0, 1, d) for d in (0, 1)] +
                  [(1, 2, d) for d in (0, 1)] + [(3, 1, 0), (4, 2, 0)],
            "c3": []}
    cubins = []
    for cfg, kernels in jobs.items():
        tmp = tempfile.mkdtemp()
        os.environ["CGF_KCACHE"] = tmp  # read per compile: one cache per config
        plan = cgf.TpPlan(config_json(cfg))
        for comp, loop, dt in kernels:
            cgf._kernel_compile(plan, comp, loop, dt)
        if cfg == "c3":  # the tcgen05 kernels of the shared-W forward / backward
            plan.compile(0, 0, True)
            plan.compile(1, 0, True)
        cubins += [(cfg, c) for c in sorted(glob.glob(os.path.join(tmp, "*.cubin")))]
    out = {}
    for cfg, cub in cubins:
        name = cfg + ":" + os.path.basename(cub).rsplit("_", 1)[0]
        sass = subprocess.run(["cuobjdump", "-sass", cub], capture_output=True, text=True).stdout
        ops = collections.Counter()
        for line in sass.splitlines():
            m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
            if m:
                ops[m.group(1).split(".")[0]] += 1
        total = sum(ops.values())
        out[name] = {"sass_instructions": total, "code_bytes": 16 * total,
                     "key_opcodes": {k: ops[k] for k in KEY if ops[k]},
                     "top": dict(ops.most_common(12))}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
