"""Benchmark: MACE-large-style uvu CG tensor product (BASELINE configs[1], "C2"),
forward + backward, FP32, batch 1M rows per GPU, on the generated sm_100a kernels.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--dtype f32|f64]
                    [--rows R] [--impl ours|reference]

One step = TP forward (z = TP(x, y, W)) + TP backward ((gx, gy, gW) from gz)
over the whole batch, inputs resident in HBM. Metric = GFLOP/s under the
reference's flop rule (kernelgen::flop_count, kernelgen.cpp:253-276):
(100,736 + 292,836) flop per row. N > 1: one process per GPU, each with its own
1M-row batch (rows are independent — "replicas / batch split"),
no data-path collective; time = max over ranks.

The line also carries "conv": the fused graph convolution of config C5 (C1 TP
on radius_graph(cubic_lattice(58^3), 3.0), 22.4M edges) as forward + backward
per step, destination-partitioned over the N ranks with NCCL all-gather of
node_x and reduce-scatter of g_node_x (paper_2501_13986_b200/dist.py);
edges/s over the whole graph, max over ranks ("scaling": "strong").

--impl reference: the reference's own CPU implementation (oracle/_ref, the
unmodified cgforge built from /root/reference) on this box's host cores, same
metric, a bounded row sample per step.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG = "c2"
HBM_FALLBACK_GBS = 6650.0


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
    ap.add_argument("--conv-n", type=int, default=58, help="lattice side of the conv leg (58 = C5); 0 = skip")
    ap.add_argument("--conv-config", default="c1", help="TP of the conv leg (C5 uses the C1 TP)")
    ap.add_argument("--conv-steps", type=int, default=5)
    ap.add_argument("--c3-rows", type=int, default=1_000_000, help="rows of the C3 (uvw, shared W) leg; 0 = skip")
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
            self._stop.wait(0.2)

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


def cpu_baseline(dtype, rows):
    """The unmodified reference (oracle/_ref) timed on this host: TpPlan
    forward + backward, all hardware threads, median of 3 after 1 warm-up
    (the CLI's methodology, tools/cgforge.cpp:336-348)."""
    from oracle import oracle as O
    if not O.ref_available():
        ref = None
    else:
        ref = O.RefPlan(O.config_json(CONFIG), budget=4096)
    import numpy as np
    dt = np.float32 if dtype == "f32" else np.float64
    cores = os.cpu_count()
    flops = (100_736 + 292_836) * rows
    if ref is not None:
        secs = ref.bench_tp(dt, rows, ops=3, warmup=1, iters=3, workers=cores)
        t = float(secs[0] + secs[1])
        kind = "reference"
    else:  # oracle port, single thread
        o = O.Oracle(O.config_json(CONFIG))
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


def run_reference(args, rank, world):
    if rank != 0:
        return
    cb = cpu_baseline(args.dtype, args.cpu_rows)
    line = {"impl": "reference", "metric": "CG TP fwd+bwd GFLOP/s (C2 MACE-large uvu)", "value": cb["value"],
            "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * (100_736 + 292_836) * args.cpu_rows / (cb["value"] * 1e9),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic (reference NormalGen inputs)",
            "config": {"workload": f"{CONFIG}: 128x0e+128x1o+128x2e x 0e+1o+2e+3o uvu, fwd+bwd",
                       "rows_per_step": args.cpu_rows},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def conv_leg(args, rank, world, dev, clk_index):
    """C5: fused conv (C1 TP) on radius_graph(cubic_lattice(n^3), 3.0),
    destination-partitioned over the ranks (dist.DistConvPlan: NCCL all-gather
    of node_x, local fused conv, reduce-scatter of g_node_x). One step =
    forward + backward, collectives included; strong scaling (|E| fixed)."""
    import torch
    import torch.distributed as dist

    import paper_2501_13986_b200 as cgf
    from paper_2501_13986_b200 import dist as cdist
    from oracle.oracle import config_json

    tdt = torch.float32 if args.dtype == "f32" else torch.float64
    es = 4 if args.dtype == "f32" else 8
    plan = cgf.TpPlan(config_json(args.conv_config))
    nodes, src, nbr = cdist.lattice_radius_graph(args.conv_n, 1.0, 3.0)
    g = cgf.Graph(nodes, src, nbr)
    del src, nbr
    sh = cdist.GraphShard(g, world, rank)
    dc = cdist.DistConvPlan(plan, sh, group=None)
    gen = torch.Generator(device=dev).manual_seed(4321 + rank)
    rnd = lambda *s: torch.randn(s, device=dev, dtype=tdt, generator=gen)
    nx, ey, ew, gnz = rnd(sh.out_nodes, plan.dim_x), rnd(sh.edges, plan.dim_y), rnd(sh.edges, plan.n_w), \
        rnd(sh.out_nodes, plan.dim_z)
    stream = torch.cuda.current_stream(dev)
    fwd_ms, bwd_ms, coll_ms = [], [], []

    def step(record=False):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(5)] if record else None
        if record:
            evs[0].record(stream)
        x_all = dc.gather_x(nx)
        if record:
            evs[1].record(stream)
        z = dc.local.forward_shard(sh, x_all, ey, ew)
        if record:
            evs[2].record(stream)
        gx_part, gy, gw = dc.local.backward_shard(sh, x_all, ey, ew, gnz)
        if record:
            evs[3].record(stream)
        gx = dc._reduce_scatter(gx_part)
        if record:
            evs[4].record(stream)
            fwd_ms.append((evs[1], evs[2]))
            bwd_ms.append((evs[2], evs[3]))
            coll_ms.append(((evs[0], evs[1]), (evs[3], evs[4])))
        return z, gx, gy, gw

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(args.conv_steps):
        step(record=True)
    b.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = torch.tensor([a.elapsed_time(b)], device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item()) / args.conv_steps
    avg = lambda L: sum(x.elapsed_time(y) for x, y in L) / len(L)
    f_ms, b_ms = avg(fwd_ms), avg(bwd_ms)
    c_ms = sum(p.elapsed_time(q) + r.elapsed_time(t) for (p, q), (r, t) in coll_ms) / len(coll_ms)
    # algorithmic bytes of this rank's kernels (SURVEY.md §8d conv rules; node
    # terms over the rows each kernel owns)
    E, Vo, Vi = sh.edges, sh.out_nodes, sh.in_nodes
    fb = (E * (plan.dim_y + plan.n_w) + Vi * plan.dim_x + Vo * plan.dim_z) * es
    bb = (2 * E * (plan.dim_y + plan.n_w) + Vi * 2 * plan.dim_x + Vo * plan.dim_z) * es
    peak, _ = measured_peak()
    per_rank = torch.tensor([f_ms, b_ms, c_ms], device=dev)
    if world > 1:
        dist.all_reduce(per_rank, op=dist.ReduceOp.MAX)
    return {
        "workload": f"c5: {args.conv_config} TP on radius_graph(cubic_lattice({args.conv_n}^3), 3.0), "
                    f"{nodes} nodes / {g.edges} edges, fwd+bwd, destination-partitioned",
        "edges_per_s": g.edges / (ms / 1e3), "ms_per_step": ms, "steps": args.conv_steps, "n_gpus": world,
        "scaling": "strong", "dtype": args.dtype,
        "collectives": "NCCL all_gather_into_tensor(node_x) + reduce_scatter_tensor(g_node_x)" if world > 1
        else "none (1 rank)",
        "max_over_ranks_ms": {"forward_kernel": float(per_rank[0]), "backward_kernel": float(per_rank[1]),
                              "collectives": float(per_rank[2])},
        "rank0_roofline": {"bound": "hbm", "peak": peak, "unit": "GB/s",
                           "forward": {"GB/s": fb / (f_ms / 1e3) / 1e9, "frac": fb / (f_ms / 1e3) / 1e9 / peak},
                           "backward": {"GB/s": bb / (b_ms / 1e3) / 1e9, "frac": bb / (b_ms / 1e3) / 1e9 / peak}},
        "gpu_launches_per_step": 2,
    }


def c3_leg(args, rank, world, dev):
    """C3: e3nn FullyConnectedTP-style uvw TP with one shared W (64x0e+64x1o+64x2e
    x 0e+1o+2e, 11 kind-C paths), FP32 forward on the tcgen05 kernel
    (3xTF32, A operand in TMEM). Per rank its own batch (replicas)."""
    import torch
    import torch.distributed as dist

    import paper_2501_13986_b200 as cgf
    from oracle.oracle import config_json

    plan = cgf.TpPlan(config_json("c3"))
    R = args.c3_rows
    g = torch.Generator(device=dev).manual_seed(99 + rank)
    x = torch.randn((R, plan.dim_x), device=dev, generator=g)
    y = torch.randn((R, plan.dim_y), device=dev, generator=g)
    w = torch.randn((1, plan.n_w), device=dev, generator=g)
    z = torch.empty((R, plan.dim_z), device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(max(3, args.warmup)):
        plan.forward(x, y, w, z=z, w_shared=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = max(3, args.steps)
    a.record(stream)
    for _ in range(steps):
        plan.forward(x, y, w, z=z, w_shared=True)
    b.record(stream)
    torch.cuda.synchronize()
    ms = torch.tensor([a.elapsed_time(b) / steps], device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    # backward on the same rows: gx (transposed forward), gz planes, gy, shared gW (+ its reduction)
    gz = torch.randn((R, plan.dim_z), device=dev, generator=g)
    outs = plan.backward(x, y, w, gz, w_shared=True)
    torch.cuda.synchronize()
    a.record(stream)
    for _ in range(steps):
        outs = plan.backward(x, y, w, gz, w_shared=True, out=outs)
    b.record(stream)
    torch.cuda.synchronize()
    bms = torch.tensor([a.elapsed_time(b) / steps], device=dev)
    if world > 1:
        dist.all_reduce(bms, op=dist.ReduceOp.MAX)
    bms = float(bms.item())
    del outs, gz
    byts = (plan.dim_x + plan.dim_y + plan.dim_z) * 4 * R + plan.n_w * 4
    peak, _ = measured_peak()
    return {"workload": "c3: 64x0e+64x1o+64x2e x 0e+1o+2e -> 64x0e+64x1o+64x2e, 11 uvw paths, shared W, fwd (+ bwd)",
            "backward_ms": bms, "backward_GFLOP/s": plan.flops_bwd * R * world / (bms / 1e3) / 1e9,
            "kernel": "cgf_uvw_fwd_f32 (tcgen05 kind::tf32, 3xTF32, A in TMEM)", "rows_per_gpu": R,
            "ms": ms, "rows_per_s": R * world / (ms / 1e3), "GFLOP/s": plan.flops_fwd * R * world / (ms / 1e3) / 1e9,
            "GB/s": byts / (ms / 1e3) / 1e9, "hbm_frac": byts / (ms / 1e3) / 1e9 / peak, "dtype": "f32"}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2501_13986_b200 as cgf
    from oracle.oracle import config_json

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    tdt = torch.float32 if args.dtype == "f32" else torch.float64
    es = 4 if args.dtype == "f32" else 8
    plan = cgf.TpPlan(config_json(CONFIG))
    R = args.rows
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    x = torch.randn((R, plan.dim_x), device=dev, dtype=tdt, generator=g)
    y = torch.randn((R, plan.dim_y), device=dev, dtype=tdt, generator=g)
    w = torch.randn((R, plan.n_w), device=dev, dtype=tdt, generator=g)
    gz = torch.randn((R, plan.dim_z), device=dev, dtype=tdt, generator=g)
    z = torch.empty((R, plan.dim_z), device=dev, dtype=tdt)
    stream = torch.cuda.current_stream(dev)

    fwd_ev, bwd_ev = [], []

    def step(record=False):
        if record:
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(stream)
        plan.forward(x, y, w, z=z)
        if record:
            e1.record(stream)
        out = plan.backward(x, y, w, gz)
        if record:
            e2.record(stream)
            fwd_ev.append((e0, e1))
            bwd_ev.append((e1, e2))
        return out

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
    ms = start.elapsed_time(stop)
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    fwd_ms = sum(a.elapsed_time(b) for a, b in fwd_ev) / len(fwd_ev)
    bwd_ms = sum(a.elapsed_time(b) for a, b in bwd_ev) / len(bwd_ev)

    flops_row = plan.flops_fwd + plan.flops_bwd
    value = flops_row * R * world * args.steps / (ms / 1e3) / 1e9
    # Algorithmic (compulsory) bytes per launch: every input read once, every
    # output written once: fwd (x+y+W+z), bwd (2x+2y+2W+z) words/row.
    fwd_bytes = (plan.dim_x + plan.dim_y + plan.n_w + plan.dim_z) * es * R
    bwd_bytes = (2 * plan.dim_x + 2 * plan.dim_y + 2 * plan.n_w + plan.dim_z) * es * R
    peak, peak_kind = measured_peak()
    kern = {"forward": {"ms": fwd_ms, "gbs": fwd_bytes / (fwd_ms / 1e3) / 1e9, "bytes": fwd_bytes},
            "backward": {"ms": bwd_ms, "gbs": bwd_bytes / (bwd_ms / 1e3) / 1e9, "bytes": bwd_bytes}}
    dom = max(kern, key=lambda k: kern[k]["ms"])
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):
        try:  # per-launch DRAM bytes of this kernel from one ncu --set full capture (tools/ncu_traffic.py)
            rec = json.load(open(tfile)).get(f"{CONFIG}_{args.dtype}_{dom}")
            traffic = None if rec is None else rec["traffic_bytes"] * R / 1_000_000
        except Exception:
            traffic = None
    roof = {"bound": "hbm", "kernel": f"cgf_tp_{'fwd' if dom == 'forward' else 'bwd'}_{args.dtype}",
            "achieved": kern[dom]["gbs"], "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
            "frac": kern[dom]["gbs"] / peak, "traffic": traffic,
            "algorithmic_bytes_per_launch": kern[dom]["bytes"],
            "per_kernel": {k: {"ms": v["ms"], "GB/s": v["gbs"], "frac": v["gbs"] / peak} for k, v in kern.items()}}

    # End to end through the public API with HOST buffers: the C ABI host
    # entry points (cgf_tp_forward_host / cgf_tp_backward_host via TpPlan on
    # numpy arrays) copy each call's inputs in and outputs back, pipelined in
    # row chunks on two streams; host wall clock around the synchronous calls.
    Re = min(args.e2e_rows, R)
    hx = x[:Re].cpu().pin_memory()
    hy = y[:Re].cpu().pin_memory()
    hw = w[:Re].cpu().pin_memory()
    hg = gz[:Re].cpu().pin_memory()
    oz = torch.empty((Re, plan.dim_z), dtype=tdt).pin_memory()
    ogx = torch.empty((Re, plan.dim_x), dtype=tdt).pin_memory()
    ogy = torch.empty((Re, plan.dim_y), dtype=tdt).pin_memory()
    ogw = torch.empty((Re, plan.n_w), dtype=tdt).pin_memory()
    nx_, ny_, nw_, ng_ = hx.numpy(), hy.numpy(), hw.numpy(), hg.numpy()
    noz, ngx, ngy, ngw = oz.numpy(), ogx.numpy(), ogy.numpy(), ogw.numpy()

    def e2e_step():
        plan.forward(nx_, ny_, nw_, z=noz)
        plan.backward(nx_, ny_, nw_, ng_, out=(ngx, ngy, ngw))

    for _ in range(2):
        e2e_step()
    if world > 1:
        dist.barrier()
    ke = max(3, args.steps // 2)
    t0 = time.perf_counter()
    for _ in range(ke):
        e2e_step()
    ems = torch.tensor([(time.perf_counter() - t0) * 1e3 / ke], device=dev)
    if world > 1:
        dist.all_reduce(ems, op=dist.ReduceOp.MAX)
    e2e_val = flops_row * Re * world / (float(ems.item()) / 1e3) / 1e9
    # bytes actually copied: forward (x, y, W in; z out) + backward (x, y, W, gz in; gx, gy, gW out)
    h2d = (2 * (hx.numel() + hy.numel() + hw.numel()) + hg.numel()) * es
    d2h = (oz.numel() + ogx.numel() + ogy.numel() + ogw.numel()) * es

    del x, y, w, gz, z, hx, hy, hw, hg, oz, ogx, ogy, ogw
    torch.cuda.empty_cache()
    c3 = None
    if args.c3_rows > 0:
        try:
            c3 = c3_leg(args, rank, world, dev)
        except Exception as exc:
            c3 = {"error": repr(exc)}
        torch.cuda.empty_cache()
    conv = None
    if args.conv_n > 0:
        try:
            conv = conv_leg(args, rank, world, dev, local)
        except Exception as exc:  # report, never sink the headline line
            conv = {"error": repr(exc)}
        torch.cuda.empty_cache()

    cb = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_baseline(args.dtype, args.cpu_rows)
        except Exception as exc:  # the baseline must never sink the GPU line
            cb = {"error": repr(exc)}

    if rank == 0:
        line = {
            "metric": "CG TP fwd+bwd GFLOP/s (C2 MACE-large uvu)", "value": value, "unit": "GFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic (torch.randn inputs of the C2 shapes)",
            "config": {"workload": "c2: 128x0e+128x1o+128x2e x 1x0e+1x1o+1x2e+1x3o -> 17 uvu paths, fwd+bwd",
                       "rows_per_gpu": R, "parallelism": f"dp{world} (independent row batches)",
                       "l2": "inputs larger than L2 (GBs per step), no flush needed",
                       "rows_per_s": R * world * args.steps / (ms / 1e3)},
            "roofline": roof,
            "cpu_baseline": cb,
            "e2e": {"value": e2e_val, "unit": "GFLOP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "rows_per_step": Re, "path": "pinned host arrays -> TpPlan.forward/backward -> cgf_tp_*_host (C ABI; chunked, 2 streams) -> pinned host", "timer": "host wall clock"},
            "gpu_launches": 2 * args.steps,  # TP leg: one forward + one backward kernel per step
            "conv": conv,
            "c3": c3,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
