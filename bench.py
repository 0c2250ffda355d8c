"""Benchmark: MACE-large-style uvu CG tensor product (BASELINE configs[1], "C2"),
forward + backward, FP32, batch 1M rows per GPU, on the generated sm_100a kernels.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--dtype f32|f64]
                    [--rows R] [--impl ours|reference]

One step = TP forward (z = TP(x, y, W)) + TP backward ((gx, gy, gW) from gz)
over the whole batch, inputs resident in HBM. Metric = GFLOP/s under the
reference's flop rule (kernelgen::flop_count, kernelgen.cpp:253-276):
(100,736 + 292,836) flop per row. N > 1: one process per GPU (the script
re-launches itself under torch.distributed.run when started without
RANK/WORLD_SIZE), each with its own 1M-row batch (rows are independent —
"replicas / batch split"), no data-path collective; time = max
over ranks.

Sub-objects of the line (each its own CUDA-event timing, max over ranks):
  conv    C5: the fused graph convolution (C1 TP on radius_graph(cubic_lattice
          (58^3), 3.0), 22.4M edges), forward + backward, destination-
          partitioned over the N ranks (NCCL all-gather of node_x, all-to-all
          + rank-ordered sum of g_node_x); edges/s over the whole graph
          ("scaling": "strong"), per-rank kernel and collective ms.
  legs    C1 (50K rows FP32 forward, BASELINE configs[0]), C2 FP64 forward /
          backward at 1M rows, C3 (uvw, shared W, tcgen05) forward / backward,
          C4 (C2 TP on the 29^3 lattice, 2.63M edges) conv forward / backward /
          double-backward in FP32 and forward / backward in FP64: ms, GB/s and
          the fraction of measured HBM per kernel.
  e2e     the same fwd+bwd step through the public API with pinned HOST
          buffers (TpPlan.forward_backward -> cgf_tp_forward_backward_host, one
          pipelined pass) with the measured PCIe roofline beside it; also the
          two separate calls (TpPlan.forward + TpPlan.backward).

--impl reference: the reference's own CPU implementation (oracle/_ref, the
unmodified cgforge built from /root/reference) on this box's host cores, same
metric, a bounded row sample per step. The in-line cpu_baseline runs the same
code in a separate process before this process touches the GPU.
"""
import argparse
import hashlib
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG = "c2"
HBM_FALLBACK_GBS = 6650.0
METRIC = "CG TP fwd+bwd GFLOP/s (C2 MACE-large uvu)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--dtype", default="f32", choices=["f32", "f64"])
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--e2e-rows", type=int, default=131_072)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-rows", type=int, default=50_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-baseline-only", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--conv-n", type=int, default=58, help="lattice side of the conv leg (58 = C5); 0 = skip")
    ap.add_argument("--conv-config", default="c1", help="TP of the conv leg (C5 uses the C1 TP)")
    ap.add_argument("--conv-steps", type=int, default=5)
    ap.add_argument("--legs", default="c1,c2f64,c3,c4", help="comma list of sub-legs; '' = none")
    ap.add_argument("--leg-steps", type=int, default=3)
    ap.add_argument("--harness-check", action="store_true",
                    help="CPU/gloo plumbing check of the multi-rank conv leg with a torch stand-in for the "
                         "kernels (numbers meaningless; never a bench value)")
    return ap.parse_args()


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------ CPU baseline --

def cpu_baseline(dtype, rows):
    """The unmodified reference (oracle/_ref) timed on this host: TpPlan
    forward + backward, all hardware threads, median of 3 after 1 warm-up
    (the CLI's methodology, tools/cgforge.cpp:336-348)."""
    from oracle import oracle as O
    from paper_2501_13986_b200.configs import config_json
    import numpy as np
    dt = np.float32 if dtype == "f32" else np.float64
    cores = os.cpu_count()
    flops = (100_736 + 292_836) * rows
    if O.ref_available():
        ref = O.RefPlan(config_json(CONFIG), budget=4096)
        secs = ref.bench_tp(dt, rows, ops=3, warmup=1, iters=3, workers=cores)
        t = float(secs[0] + secs[1])
        kind = "reference"
    else:  # oracle port, single thread
        o = O.Oracle(config_json(CONFIG))
        x, y, w = O.random_batch(o, rows, 1234, dt)
        gz = O.NormalGen(1235).normal_vec(rows * o.dim_z, dt).reshape(rows, -1)
        t0 = time.perf_counter()
        o.forward(x, y, w)
        o.backward(x, y, w, gz)
        t = time.perf_counter() - t0
        kind, cores = "port", 1
    return {"value": flops / t / 1e9, "unit": "GFLOP/s", "cores": cores, "kind": kind,
            "sample": f"{CONFIG} {dtype} fwd+bwd, {rows} rows (reference random_batch inputs), "
                      f"median of 3 after 1 warm-up, {t:.3f} s per fwd+bwd",
            "rows_per_s": rows / t}


def cpu_baseline_subprocess(args):
    """cpu_baseline in a fresh process, before this one initialises CUDA (no
    GPU-side threads or pinned-memory traffic competing for the host cores)."""
    p = subprocess.run([sys.executable, os.path.abspath(__file__), "--cpu-baseline-only", "--dtype", args.dtype,
                        "--cpu-rows", str(args.cpu_rows)], capture_output=True, text=True, timeout=900)
    if p.returncode != 0:
        return {"error": (p.stderr or p.stdout)[-400:]}
    rec = json.loads(p.stdout.strip().splitlines()[-1])
    rec["process"] = "separate, before CUDA init"
    return rec


def run_reference(args, rank, world):
    if rank != 0:
        return
    cb = cpu_baseline(args.dtype, args.cpu_rows)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"],
            "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * (100_736 + 292_836) * args.cpu_rows / (cb["value"] * 1e9),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic (reference NormalGen inputs)",
            "config": {"workload": f"{CONFIG}: 128x0e+128x1o+128x2e x 0e+1o+2e+3o uvu, fwd+bwd",
                       "rows_per_step": args.cpu_rows},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------- helpers ----

def event_ms(fn, steps, stream):
    """Average device ms of fn() over `steps` back-to-back calls (CUDA events
    on the launching stream, synchronised on both sides)."""
    import torch
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def max_over_ranks(vals, dev, world):
    import torch
    import torch.distributed as dist
    t = torch.tensor(vals, device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.tolist()]


def kernel_source_sha(plan, op, dtype_code):
    import paper_2501_13986_b200 as cgf
    return hashlib.sha256(plan.source(op, dtype_code).encode()).hexdigest()[:16]


def ncu_traffic(key, src_sha, R):
    """Per-launch DRAM bytes of this kernel from the committed `ncu --set full`
    capture (profiles/ncu_traffic.json, tools/ncu_traffic.py), scaled to R rows;
    None unless the capture was taken of the same generated kernel source."""
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        rec = json.load(open(tfile)).get(key)
    except Exception:
        return None, "no capture"
    if rec is None:
        return None, "no capture"
    if rec.get("source_sha16") != src_sha:
        return None, f"stale capture (kernel source {rec.get('source_sha16')} != {src_sha})"
    return rec["traffic_bytes"] * R / rec.get("rows", 1_000_000), rec.get("report")


def measure_pcie(dev, gib=1.0):
    """Pinned host <-> device copy bandwidth (GB/s): H2D alone, D2H alone and
    both directions at once (two streams) — the ceiling of the e2e path."""
    import torch
    n = int(gib * (1 << 30)) // 4
    h1 = torch.empty(n, dtype=torch.float32).pin_memory()
    h2 = torch.empty(n, dtype=torch.float32).pin_memory()
    d1 = torch.empty(n, dtype=torch.float32, device=dev)
    d2 = torch.empty(n, dtype=torch.float32, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    nbytes = 4 * n

    def timed(do_h2d, do_d2h, reps=3):
        best = float("inf")
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if do_h2d:
                with torch.cuda.stream(s1):
                    d1.copy_(h1, non_blocking=True)
            if do_d2h:
                with torch.cuda.stream(s2):
                    h2.copy_(d2, non_blocking=True)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        return best

    timed(True, True, 1)
    h2d = nbytes / timed(True, False) / 1e9
    d2h = nbytes / timed(False, True) / 1e9
    both = 2 * nbytes / timed(True, True) / 1e9
    del h1, h2, d1, d2
    return {"h2d_GBps": h2d, "d2h_GBps": d2h, "bidirectional_GBps": both,
            "how": f"pinned torch copies of {gib:g} GiB, best of 3, host wall clock"}


# ------------------------------------------------------------ legs ---------

def tp_leg(cgf, plan, name, R, dtype, ops, steps, dev, world, w_shared=False, peak=None):
    """Device-resident TP ops on R rows (torch.randn inputs), CUDA events per
    op; algorithmic bytes from cgf_tp_traffic (each input read once, each
    output written once)."""
    import torch
    tdt = torch.float32 if dtype == "f32" else torch.float64
    es = 4 if dtype == "f32" else 8
    g = torch.Generator(device=dev).manual_seed(7)
    x = torch.randn((R, plan.dim_x), device=dev, dtype=tdt, generator=g)
    y = torch.randn((R, plan.dim_y), device=dev, dtype=tdt, generator=g)
    w = torch.randn((1 if w_shared else R, plan.n_w), device=dev, dtype=tdt, generator=g)
    zbuf = torch.randn((R, plan.dim_z), device=dev, dtype=tdt, generator=g)  # z of the forward, gz of the backward
    stream = torch.cuda.current_stream(dev)
    out = {"workload": name, "rows": R, "dtype": dtype}
    bwd_out = None
    for op in ops:
        if op == "forward":
            fn = lambda: plan.forward(x, y, w, z=zbuf, w_shared=w_shared)
            code = 0
        else:
            if bwd_out is None:
                bwd_out = plan.backward(x, y, w, zbuf, w_shared=w_shared)
            fn = lambda: plan.backward(x, y, w, zbuf, w_shared=w_shared, out=bwd_out)
            code = 1
        fn()
        ms = max_over_ranks([event_ms(fn, steps, stream)], dev, world)[0]
        words = sum(plan.traffic(code, R, w_shared))
        gbs = words * es / (ms / 1e3) / 1e9
        flops = (plan.flops_fwd if code == 0 else plan.flops_bwd) * R
        out[op] = {"ms": ms, "GB/s": gbs, "hbm_frac": gbs / peak, "GFLOP/s": flops / (ms / 1e3) / 1e9,
                   "algorithmic_bytes": words * es}
    del x, y, w, zbuf, bwd_out
    torch.cuda.empty_cache()
    return out


# tcgen05 kind::tf32 peak measured on this part by tools/tc_bench.cu
# (profiles/r01_tc_bench.log: M=128, N=128, K=8 MMAs, 2046 MAC / cycle / SM)
TF32_MAC_PER_CLK_SM = 2046
SM_COUNT = 148


def uvw_mma_flops_per_row(cfg_name):
    """Dense W contraction flops per row of a kind-C problem (sum over
    instructions of 2 * (2 l3 + 1) * b * b'), from its problem JSON."""
    from paper_2501_13986_b200.configs import CONFIGS
    js = CONFIGS[cfg_name]
    seg = lambda s: [(int(t.split("x")[0]), int(t.split("x")[1][:-1])) for t in s.replace(" ", "").split("+")]
    X, Z = seg(js["x"]), seg(js["z"])
    return sum(2 * (2 * Z[zs - 1][1] + 1) * Z[zs - 1][0] * X[xs - 1][0] for xs, _, zs, _ in js["instructions"])


def tensor_roofline(ms, mma_flops, clk_mhz):
    """3xTF32 tensor-core work (3 MMAs per product) against the measured tf32 peak."""
    peak = TF32_MAC_PER_CLK_SM * 2 * SM_COUNT * clk_mhz * 1e6 / 1e12
    achieved = 3 * mma_flops / (ms / 1e3) / 1e12
    return {"bound": "tensor", "unit": "TFLOP/s", "achieved": achieved, "peak": peak, "frac": achieved / peak,
            "peak_kind": f"measured tf32 MMA rate (tools/tc_bench.cu) at {clk_mhz:.0f} MHz",
            "mma_flops_per_launch": 3 * mma_flops}


def conv_single_leg(cgf, cdist, name, tp_name, n, dtypes_ops, steps, dev, peak):
    """Fused conv on one GPU (C4: C2 TP on radius_graph(cubic_lattice(n^3), 3.0))."""
    import torch
    from paper_2501_13986_b200.configs import config_json
    plan = cgf.TpPlan(config_json(tp_name))
    cp = cgf.ConvPlan(plan)
    nodes, src, nbr = cdist.lattice_radius_graph(n, 1.0, 3.0)
    g = cgf.Graph(nodes, src, nbr)
    del src, nbr
    E, V = g.edges, g.nodes
    stream = torch.cuda.current_stream(dev)
    out = {"workload": f"{name}: {tp_name} TP on radius_graph(cubic_lattice({n}^3), 3.0), {V} nodes / {E} edges",
           "nodes": V, "edges": E}
    dyw = plan.dim_y + plan.n_w
    words = {"forward": E * dyw + V * (plan.dim_x + plan.dim_z),
             "backward": 2 * E * dyw + V * (2 * plan.dim_x + plan.dim_z),
             "double_backward": 3 * E * dyw + V * (3 * plan.dim_x + 2 * plan.dim_z)}
    flops = {"forward": plan.flops_fwd, "backward": plan.flops_bwd, "double_backward": plan.flops_dbwd}
    for dtype, ops in dtypes_ops:
        tdt = torch.float32 if dtype == "f32" else torch.float64
        es = 4 if dtype == "f32" else 8
        gen = torch.Generator(device=dev).manual_seed(11)
        rnd = lambda *s: torch.randn(s, device=dev, dtype=tdt, generator=gen)
        nx, ey, ew, gnz = rnd(V, plan.dim_x), rnd(E, plan.dim_y), rnd(E, plan.n_w), rnd(V, plan.dim_z)
        res = {}
        for op in ops:
            if op == "forward":
                fn = lambda: cp.forward(g, nx, ey, ew)
            elif op == "backward":
                fn = lambda: cp.backward(g, nx, ey, ew, gnz)
            else:
                up = (rnd(V, plan.dim_x), rnd(E, plan.dim_y), rnd(E, plan.n_w))
                fn = lambda: cp.double_backward(g, nx, ey, ew, gnz, up)
            r = fn()
            del r
            ms = event_ms(fn, steps, stream)
            gbs = words[op] * es / (ms / 1e3) / 1e9
            res[op] = {"ms": ms, "GB/s": gbs, "hbm_frac": gbs / peak, "edges_per_s": E / (ms / 1e3),
                       "GFLOP/s": flops[op] * E / (ms / 1e3) / 1e9}
            if op == "double_backward":
                del up
            torch.cuda.empty_cache()
        out[dtype] = res
        del nx, ey, ew, gnz
        torch.cuda.empty_cache()
    return out


class _TorchShardStandIn:
    """--harness-check only: stands in for the CUDA shard kernels on CPU ranks
    (a linear map of the gathered neighbour rows), so the multi-rank plumbing
    — partition, all-gather, all-to-all reduction, timing, max over ranks,
    the JSON line — runs under gloo. Its numbers are not a measurement."""

    def __init__(self, plan):
        self.plan = plan

    def forward_shard(self, sh, x_all, ey, ew, mode=0, rows=None, out=None):
        import torch
        d = sh.device(x_all.device)
        src = torch.repeat_interleave(torch.arange(sh.out_nodes), d["row_ptr"].diff())
        z = x_all.new_zeros((sh.out_nodes, self.plan.dim_z))
        z[:, :self.plan.dim_x].index_add_(0, src, x_all[d["nbr"].long()])
        if rows is None:
            return z
        out = x_all.new_zeros(z.shape) if out is None else out
        out[rows[0]:rows[1]] = z[rows[0]:rows[1]]
        return out

    def backward_shard(self, sh, x_all, ey, ew, gz, mode=0, rows=None, outs=None):
        import torch
        d = sh.device(x_all.device)
        src = torch.repeat_interleave(torch.arange(sh.out_nodes), d["row_ptr"].diff())
        gx = x_all.new_zeros((sh.in_nodes, self.plan.dim_x))
        gx.index_add_(0, d["nbr"].long(), gz[src, :self.plan.dim_x])
        if rows is None:
            return gx, torch.zeros_like(ey), torch.zeros_like(ew)
        outs = (x_all.new_zeros(gx.shape), torch.zeros_like(ey), torch.zeros_like(ew)) if outs is None else outs
        outs[0][rows[0]:rows[1]] = gx[rows[0]:rows[1]]
        return outs


def conv_leg(args, rank, world, dev, harness=False):
    """C5: fused conv (C1 TP) on radius_graph(cubic_lattice(n^3), 3.0),
    destination-partitioned over the ranks (dist.DistConvPlan: NCCL all-gather
    of node_x, local fused conv, all-to-all + rank-ordered sum of g_node_x).
    One step = forward + backward, collectives included; strong scaling (|E|
    fixed)."""
    import torch
    import torch.distributed as dist

    import paper_2501_13986_b200 as cgf
    from paper_2501_13986_b200 import dist as cdist
    from paper_2501_13986_b200.configs import config_json

    tdt = torch.float32 if args.dtype == "f32" else torch.float64
    es = 4 if args.dtype == "f32" else 8
    plan = cgf.TpPlan(config_json(args.conv_config))
    nodes, src, nbr = cdist.lattice_radius_graph(args.conv_n, 1.0, 3.0)
    g = cgf.Graph(nodes, src, nbr)
    del src, nbr
    sh = cdist.GraphShard(g, world, rank)
    dc = cdist.DistConvPlan(plan, sh, group=None, local=_TorchShardStandIn(plan) if harness else None)
    gen = torch.Generator(device=dev).manual_seed(4321 + rank)
    rnd = lambda *s: torch.randn(s, device=dev, dtype=tdt, generator=gen)
    nx, ey, ew, gnz = rnd(sh.out_nodes, plan.dim_x), rnd(sh.edges, plan.dim_y), rnd(sh.edges, plan.n_w), \
        rnd(sh.out_nodes, plan.dim_z)
    cuda = dev.type == "cuda"
    stream = torch.cuda.current_stream(dev) if cuda else None
    laps = []

    def mark():
        if cuda:
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            return e
        return time.perf_counter()

    def lap(a, b):
        return a.elapsed_time(b) if cuda else (b - a) * 1e3

    def step(record=False):
        # unoverlapped: all-gather | forward kernel | backward kernel | exchange + ordered sum
        t0 = mark()
        x_all = dc.gather_x(nx)
        t1 = mark()
        z = dc.local.forward_shard(sh, x_all, ey, ew)
        t2 = mark()
        gx_part, gy, gw = dc.local.backward_shard(sh, x_all, ey, ew, gnz)
        t3 = mark()
        gx = dc._reduce_scatter(gx_part)
        t4 = mark()
        if record:
            laps.append((t0, t1, t2, t3, t4))
        return z, gx, gy, gw

    def step_overlap(record=False):
        # overlapped (DistConvPlan default at N > 1): local-neighbour rows run
        # during the all-gather, own neighbour rows during the exchange
        t0 = mark()
        z, x_all = dc.forward_gathered(nx, ey, ew)
        t1 = mark()
        gx, gy, gw = dc.backward(nx, ey, ew, gnz, node_x_all=x_all)
        t2 = mark()
        if record:
            laps.append((t0, t1, t2))
        return z, gx, gy, gw

    def timed(fn):
        laps.clear()
        for _ in range(max(3, args.warmup)):
            fn()
        if cuda:
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        if cuda:
            torch.cuda.synchronize()
        a = mark()
        for _ in range(args.conv_steps):
            fn(record=True)
        b = mark()
        if cuda:
            torch.cuda.synchronize()
        return lap(a, b) / args.conv_steps, [sum(lap(t[i], t[i + 1]) for t in laps) / len(laps)
                                             for i in range(len(laps[0]) - 1)]

    ms, (ag_ms, f_ms, b_ms, rs_ms) = timed(step)
    ov_err = None
    try:
        ov_ms, ov_f, ov_b = (ms, f_ms + ag_ms, b_ms + rs_ms) if world == 1 else (lambda r: (r[0], *r[1]))(
            timed(step_overlap))
    except Exception as exc:  # keep the unoverlapped measurement if the overlapped path fails
        ov_err = repr(exc)[:300]
        ov_ms, ov_f, ov_b = ms, f_ms + ag_ms, b_ms + rs_ms
    t = torch.tensor([ms, f_ms, b_ms, ag_ms, rs_ms, ov_ms, ov_f, ov_b], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, f_mx, b_mx, ag_mx, rs_mx, ov_mx, ovf_mx, ovb_mx = (float(v) for v in t.tolist())
    unoverlapped_ms = ms
    ms = ov_mx  # the DistConvPlan default (overlapped at N > 1; the same step at N = 1)
    E, Vo, Vi = sh.edges, sh.out_nodes, sh.in_nodes
    fb = (E * (plan.dim_y + plan.n_w) + Vi * plan.dim_x + Vo * plan.dim_z) * es
    bb = (2 * E * (plan.dim_y + plan.n_w) + Vi * 2 * plan.dim_x + Vo * plan.dim_z) * es
    peak, _ = measured_peak()
    return {
        "workload": f"c5: {args.conv_config} TP on radius_graph(cubic_lattice({args.conv_n}^3), 3.0), "
                    f"{nodes} nodes / {g.edges} edges, fwd+bwd, destination-partitioned",
        "edges_per_s": g.edges / (ms / 1e3), "ms_per_step": ms, "steps": args.conv_steps, "n_gpus": world,
        "scaling": "strong", "dtype": args.dtype,
        "collectives": "in-place all_gather_into_tensor(node_x) overlapped with the local-neighbour rows; "
                       "point-to-point exchange of g_node_x partials overlapped with the own neighbour rows; "
                       "rank-ordered sum (step_unoverlapped: all_to_all_single after the kernels)"
        if world > 1 else "none (1 rank)",
        "max_over_ranks_ms": {"step": ms, "forward_kernel": f_mx, "backward_kernel": b_mx,
                              "all_gather": ag_mx, "reduce": rs_mx, "step_unoverlapped": unoverlapped_ms,
                              "step_overlapped": ov_mx, "forward_with_all_gather_overlapped": ovf_mx,
                              "backward_with_exchange_overlapped": ovb_mx},
        "overlap": {"local_rows": list(sh.local_rows()), "own_neighbour_rows": list(sh.own_rows()),
                    "out_nodes": sh.out_nodes, "in_nodes": sh.in_nodes, "error": ov_err} if world > 1 else None,
        "rank0_roofline": {"bound": "hbm", "peak": peak, "unit": "GB/s",
                           "forward": {"GB/s": fb / (f_ms / 1e3) / 1e9, "frac": fb / (f_ms / 1e3) / 1e9 / peak},
                           "backward": {"GB/s": bb / (b_ms / 1e3) / 1e9, "frac": bb / (b_ms / 1e3) / 1e9 / peak}},
        "gpu_launches_per_step": 2,
    }


def harness_check(args):
    """CPU / gloo run of the multi-rank conv leg with the torch stand-in."""
    import torch
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        dist.init_process_group("gloo")
    conv = conv_leg(args, rank, world, torch.device("cpu"), harness=True)
    if rank == 0:
        print(json.dumps({"harness": True, "n_gpus": world, "conv": conv}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def respawn(args):
    """`--gpus N` without a torch.distributed environment: re-launch this
    script as N ranks (one per GPU) under torch.distributed.run."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ---------------------------------------------------------------- main -----

def main():
    args = parse()
    if args.cpu_baseline_only:
        print(json.dumps(cpu_baseline(args.dtype, args.cpu_rows)), flush=True)
        return 0
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return respawn(args)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if args.harness_check:
        return harness_check(args)

    # the CPU baseline first, in its own process, before CUDA is initialised here
    cb = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_baseline_subprocess(args)
        except Exception as exc:  # the baseline must never sink the GPU line
            cb = {"error": repr(exc)}

    import torch
    import torch.distributed as dist

    import paper_2501_13986_b200 as cgf
    from paper_2501_13986_b200 import dist as cdist
    from paper_2501_13986_b200.configs import config_json

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    tdt = torch.float32 if args.dtype == "f32" else torch.float64
    es = 4 if args.dtype == "f32" else 8
    dcode = cgf.F32 if args.dtype == "f32" else cgf.F64
    peak, peak_kind = measured_peak()
    plan = cgf.TpPlan(config_json(CONFIG))
    R = args.rows
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    x = torch.randn((R, plan.dim_x), device=dev, dtype=tdt, generator=g)
    y = torch.randn((R, plan.dim_y), device=dev, dtype=tdt, generator=g)
    w = torch.randn((R, plan.n_w), device=dev, dtype=tdt, generator=g)
    gz = torch.randn((R, plan.dim_z), device=dev, dtype=tdt, generator=g)
    z = torch.empty((R, plan.dim_z), device=dev, dtype=tdt)
    grads = plan.backward(x, y, w, gz)
    stream = torch.cuda.current_stream(dev)

    fwd_ev, bwd_ev = [], []

    def step(record=False):
        if record:
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(stream)
        plan.forward(x, y, w, z=z)
        if record:
            e1.record(stream)
        plan.backward(x, y, w, gz, out=grads)
        if record:
            e2.record(stream)
            fwd_ev.append((e0, e1))
            bwd_ev.append((e1, e2))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        start.record(stream)
        for _ in range(args.steps):
            step(record=True)
        stop.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    fwd_ms = sum(a.elapsed_time(b) for a, b in fwd_ev) / len(fwd_ev)
    bwd_ms = sum(a.elapsed_time(b) for a, b in bwd_ev) / len(bwd_ev)
    ms, fwd_ms, bwd_ms = max_over_ranks([start.elapsed_time(stop), fwd_ms, bwd_ms], dev, world)

    flops_row = plan.flops_fwd + plan.flops_bwd
    value = flops_row * R * world * args.steps / (ms / 1e3) / 1e9
    # Algorithmic (compulsory) bytes per launch: every input read once, every
    # output written once: fwd (x+y+W+z), bwd (2x+2y+2W+z) words/row.
    fwd_bytes = sum(plan.traffic(cgf.OP_FORWARD, R)) * es
    bwd_bytes = sum(plan.traffic(cgf.OP_BACKWARD, R)) * es
    kern = {"forward": {"ms": fwd_ms, "gbs": fwd_bytes / (fwd_ms / 1e3) / 1e9, "bytes": fwd_bytes, "op": 0},
            "backward": {"ms": bwd_ms, "gbs": bwd_bytes / (bwd_ms / 1e3) / 1e9, "bytes": bwd_bytes, "op": 1}}
    dom = max(kern, key=lambda k: kern[k]["ms"])
    kname = f"cgf_tp_{'fwd' if dom == 'forward' else 'bwd'}_{args.dtype}"
    src_sha = kernel_source_sha(plan, kern[dom]["op"], dcode)
    traffic, traffic_src = ncu_traffic(f"{CONFIG}_{args.dtype}_{dom}", src_sha, R)
    roof = {"bound": "hbm", "kernel": kname, "achieved": kern[dom]["gbs"], "peak": peak, "peak_kind": peak_kind,
            "unit": "GB/s", "frac": kern[dom]["gbs"] / peak, "traffic": traffic, "traffic_source": traffic_src,
            "kernel_source_sha16": src_sha, "algorithmic_bytes_per_launch": kern[dom]["bytes"],
            "per_kernel": {k: {"ms": v["ms"], "GB/s": v["gbs"], "frac": v["gbs"] / peak} for k, v in kern.items()}}
    del x, y, w, gz, z, grads
    torch.cuda.empty_cache()

    # ---- end to end through the public API with HOST buffers --------------
    pcie = measure_pcie(dev)
    # per rank; halved beyond 2 ranks so N ranks' pinned buffers (13 GB each
    # at 131,072 rows) stay well inside the host's memory
    Re = args.e2e_rows if world <= 2 else args.e2e_rows // 2
    gh = torch.Generator().manual_seed(99 + rank)
    pin = lambda *s: torch.randn(s, dtype=tdt, generator=gh).pin_memory()
    hx, hy, hw, hg = pin(Re, plan.dim_x), pin(Re, plan.dim_y), pin(Re, plan.n_w), pin(Re, plan.dim_z)
    outs = [torch.empty(s, dtype=tdt).pin_memory() for s in
            ((Re, plan.dim_z), (Re, plan.dim_x), (Re, plan.dim_y), (Re, plan.n_w))]
    nin = [a.numpy() for a in (hx, hy, hw, hg)]
    nout = tuple(a.numpy() for a in outs)

    def e2e_fused():
        plan.forward_backward(*nin, out=nout)

    def e2e_separate():
        plan.forward(nin[0], nin[1], nin[2], z=nout[0])
        plan.backward(*nin, out=nout[1:])

    e2e = {}
    ke = max(3, args.steps // 2)
    for name, fn in (("fused", e2e_fused), ("separate", e2e_separate)):
        for _ in range(2):
            fn()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(ke):
            fn()
        e2e[name] = max_over_ranks([(time.perf_counter() - t0) * 1e3 / ke], dev, world)[0]
    in_b = sum(a.numel() for a in (hx, hy, hw, hg)) * es
    out_b = sum(a.numel() for a in outs) * es
    sep_h2d = in_b + (hx.numel() + hy.numel() + hw.numel()) * es  # the backward re-uploads x, y, W
    e2e_val = flops_row * Re * world / (e2e["fused"] / 1e3) / 1e9
    pcie_bound_ms = max(in_b / pcie["h2d_GBps"], out_b / pcie["d2h_GBps"],
                        (in_b + out_b) / pcie["bidirectional_GBps"]) / 1e6
    e2e_line = {"value": e2e_val, "unit": "GFLOP/s", "h2d_bytes_per_step": in_b, "d2h_bytes_per_step": out_b,
                "rows_per_step": Re, "ms_per_step": e2e["fused"],
                "path": "pinned host arrays -> TpPlan.forward_backward -> cgf_tp_forward_backward_host (C ABI; "
                        "row chunks pipelined on 3 streams: H2D | fwd+bwd kernels | D2H) -> pinned host",
                "timer": "host wall clock, max over ranks",
                "pcie": pcie, "pcie_bound_ms": pcie_bound_ms, "pcie_frac": pcie_bound_ms / e2e["fused"],
                "separate_calls": {"value": flops_row * Re * world / (e2e["separate"] / 1e3) / 1e9,
                                   "ms_per_step": e2e["separate"], "h2d_bytes_per_step": sep_h2d,
                                   "d2h_bytes_per_step": out_b,
                                   "path": "TpPlan.forward then TpPlan.backward (cgf_tp_forward_host, "
                                           "cgf_tp_backward_host)"}}
    del hx, hy, hw, hg, outs, nin, nout
    torch.cuda.empty_cache()

    # ---- sub-legs ------------------------------------------------------------
    legs = {}
    # the sub-legs are per-GPU replicas: measured at N = 1 only (at N > 1 a
    # failure on one rank inside a leg's collective would stall the others)
    want = [s for s in args.legs.split(",") if s] if world == 1 else []
    ls = args.leg_steps

    def run_leg(name, fn):
        try:
            legs[name] = fn()
        except Exception as exc:  # report, never sink the headline line
            legs[name] = {"error": repr(exc)[:400]}
        torch.cuda.empty_cache()

    if "c1" in want:
        c1 = cgf.TpPlan(config_json("c1"))
        run_leg("c1", lambda: tp_leg(cgf, c1, "c1: 32x0e+32x1o+32x2e x 0e+1o+2e, 15 uvu paths (BASELINE configs[0])",
                                     50_000, "f32", ("forward", "backward"), max(20, ls), dev, world, peak=peak))
    if "c2f64" in want:
        run_leg("c2_f64", lambda: tp_leg(cgf, plan, "c2 FP64", 1_000_000, "f64", ("forward", "backward"), ls, dev,
                                         world, peak=peak))
    if "c3" in want:
        c3 = cgf.TpPlan(config_json("c3"))
        run_leg("c3", lambda: tp_leg(cgf, c3, "c3: 64x0e+64x1o+64x2e x 0e+1o+2e, 11 uvw paths, shared W "
                                              "(tcgen05 kind::tf32, 3xTF32)", 1_000_000, "f32",
                                     ("forward", "backward"), ls, dev, world, w_shared=True, peak=peak))
        try:
            mf = uvw_mma_flops_per_row("c3") * 1_000_000
            mhz = clk.summary().get("sm_mhz") or 1965.0
            legs["c3"]["forward"]["tensor_roofline"] = tensor_roofline(legs["c3"]["forward"]["ms"], mf, mhz)
            # backward: gx (the transposed forward), gzp = gz W (gy) and the rows-contracted gW, 3x the forward's MMAs
            legs["c3"]["backward"]["tensor_roofline"] = tensor_roofline(legs["c3"]["backward"]["ms"], 3 * mf, mhz)
        except Exception as exc:  # never sink the line
            legs.setdefault("c3", {})["tensor_roofline_error"] = repr(exc)[:200]
    if "c4" in want and world == 1:
        run_leg("c4", lambda: conv_single_leg(cgf, cdist, "c4", "c2", 29,
                                              (("f32", ("forward", "backward", "double_backward")),
                                               ("f64", ("forward", "backward"))), ls, dev, peak))
    conv = None
    if args.conv_n > 0:
        try:
            conv = conv_leg(args, rank, world, dev)
        except Exception as exc:  # report, never sink the headline line
            conv = {"error": repr(exc)[:400]}
        torch.cuda.empty_cache()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic (torch.randn inputs of the C2 shapes)",
            "config": {"workload": "c2: 128x0e+128x1o+128x2e x 1x0e+1x1o+1x2e+1x3o -> 17 uvu paths, fwd+bwd",
                       "rows_per_gpu": R, "parallelism": f"dp{world} (independent row batches)",
                       "l2": "inputs larger than L2 (GBs per step), no flush needed",
                       "rows_per_s": R * world * args.steps / (ms / 1e3)},
            "roofline": roof,
            "cpu_baseline": cb,
            "e2e": e2e_line,
            "gpu_launches": 2 * args.steps,  # TP leg: one forward + one backward kernel per step
            "conv": conv,
            "legs": legs,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main() or 0)
