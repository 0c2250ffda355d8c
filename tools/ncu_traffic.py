"""Extracts per-launch DRAM traffic and duration of the captured kernels
(gpurun_out/full_*.ncu-rep) into profiles/ncu_traffic.json, the `traffic`
source of bench.py's roofline object. Each record carries the sha256 (16 hex)
of the generated kernel source it was captured from; bench.py uses a record
only when the kernel it times has the same source (otherwise "stale").

    python tools/ncu_traffic.py [gpurun_out]"""
import csv
import glob
import json
import os
import subprocess
import sys

import hashlib

d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root)
import paper_2501_13986_b200 as cgf  # noqa: E402
from paper_2501_13986_b200.configs import config_json  # noqa: E402


def source_sha(cfg, dtype, op, w_shared):
    plan = cgf.TpPlan(config_json(cfg))
    src = plan.source(0 if op == "fwd" else 1, 0 if dtype == "f32" else 1, w_shared)
    return hashlib.sha256(src.encode()).hexdigest()[:16]



out = {}
for rep in sorted(glob.glob(os.path.join(d, "full_*.ncu-rep"))):
    key = os.path.basename(rep)[5:-8]  # e.g. c2_f32_bwd
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    if len(rows) < 3:
        continue
    h, units, v = rows[0], rows[1], rows[2]
    get = lambda k: (float(v[h.index(k)].replace(",", "")), units[h.index(k)])

    def to_bytes(val, unit):
        return val * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)

    rd, wr = to_bytes(*get("dram__bytes_read.sum")), to_bytes(*get("dram__bytes_write.sum"))
    t, tu = get("gpu__time_duration.sum")
    t_ms = t * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(tu, 1)
    name = v[h.index("Kernel Name")]
    op = {"fwd": "forward", "bwd": "backward"}.get(key.split("_")[-1])
    if op is None:  # not a bench kernel capture (e.g. an A/B variant)
        continue
    cfg, dtype, opk = key.split("_")[:3]
    out[key.rsplit("_", 1)[0] + "_" + op] = {"kernel": name, "dram_read_bytes": rd, "dram_write_bytes": wr,
                                              "traffic_bytes": rd + wr, "ncu_ms": t_ms, "rows": 1_000_000,
                                              "source_sha16": source_sha(cfg, dtype, opk, cfg == "c3"),
                                              "report": os.path.basename(rep)}
path = os.path.join(root, "profiles", "ncu_traffic.json")
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out, indent=1))
