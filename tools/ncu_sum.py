"""Summarise an ncu report (raw page) into the metrics we track: time, DRAM
bytes, occupancy limits, issue activity and the dominant stall reasons.

    python tools/ncu_sum.py gpurun_out/prof.ncu-rep
"""
import csv
import subprocess
import sys

WANT = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'launch__shared_mem_per_block_dynamic', 'smsp__inst_executed.sum',
        'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'launch__grid_size', 'launch__block_size',
        'lts__t_sector_hit_rate.pct', 'l1tex__t_sector_hit_rate.pct', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    hdr, units = r[0], r[1]
    res = []
    for row in r[2:]:
        d = {}
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                d[w] = (row[i], units[i])
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith('smsp__average_warps_issue_stalled_') and h.endswith('_per_issue_active.ratio'):
                try:
                    v = float(row[i])
                except ValueError:
                    continue
                if v >= 0.05:
                    stalls.append((v, h[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]))
        d['stalls'] = sorted(stalls, reverse=True)
        res.append(d)
    return res


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        for d in summarise(rep):
            print("-----", rep)
            for k, v in d.items():
                if k == 'stalls':
                    print("  stalls (warps per issue):", ", ".join(f"{n} {x:.2f}" for x, n in v[:8]))
                else:
                    print("  %-62s %s %s" % (k[:62], v[0][:90], v[1]))
