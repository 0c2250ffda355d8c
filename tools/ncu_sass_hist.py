"""Executed SASS instructions and stall samples of an ncu report, grouped by
opcode (ncu --page source --print-source sass): where a kernel's issue slots
and stalls go.

    python tools/ncu_sass_hist.py gpurun_out/full_x.ncu-rep [per_unit_divisor]
"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr = next(r for r in rows if "Address" in r)
i_src, i_exe, i_smp = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
exe, smp = collections.Counter(), collections.Counter()
for r in rows[rows.index(hdr) + 1:]:
    if len(r) <= i_exe or not r[i_exe].replace(".", "").isdigit():
        continue
    toks = r[i_src].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    op = op.split(".")[0]
    exe[op] += float(r[i_exe])
    smp[op] += float(r[i_smp] or 0)
te, ts = sum(exe.values()), sum(smp.values())
print(f"{rep}: {te:.4g} warp instructions executed ({te / div:.1f} per unit), {ts:.0f} stall samples")
for op, n in exe.most_common(25):
    print(f"  {op:10s} {n / div:10.1f} /unit  {100 * n / te:5.1f} % of issue   {100 * smp[op] / max(ts, 1):5.1f} % of stall samples")
