"""Benchmark of the IOS stage executor (BASELINE.json metric: batch-1 latency ms of the IOS schedule
vs the sequential and greedy schedules on the same kernels, + % of per-stage roofline).

python bench.py [--gpus N] [--steps K] [--warmup W] [--net inception_v3] [--impl ours|reference]

One step = one inference of the whole network through ios_run (every stage of Q, one launch each,
captured in a CUDA graph), inputs resident in HBM; L2 is flushed (a 2x-L2 write) before every timed
step. N > 1 (`--gpus N`; re-executed under torch.distributed.run when launched directly): one
process per GPU, the global batch (default 8 per GPU) sharded by image, each rank its own graph and
DP schedule, no collective on the hot path, device time max over ranks.
`--impl reference` times the CPU oracle (the tier's reference arm) on a bounded sample of the
same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NETS = {
    "inception_v3": dict(math="tf32", desc="Inception V3 batch 1, 299x299, TF32 on 1xB200"),
    "nasnet_a_large": dict(math="tf32", desc="NasNet-A large batch 1, 331x331, TF32"),
    "randwire_ws_small": dict(math="bf16", desc="RandWire-WS small batch 1, 224x224, BF16"),
    "squeezenet": dict(math="tf32", desc="SqueezeNet v1.0 224x224, TF32"),
    "fig2": dict(math="tf32", desc="Fig.2 4-conv block 1x64x28x28, TF32"),
}
METRIC = "batch-1 latency ms (IOS vs sequential/greedy schedule) + % stage roofline"


def _peaks(measure_tf32: bool = False, device=None):
    """Roofline denominators: MEASURED_PEAKS.json (driver-written HBM copy GB/s and cuBLAS bf16 TF/s on
    this pool's B200s) and, when a GPU is at hand, the dense TF32 peak measured here (cuBLAS fp32
    matmul with allow_tf32, best of 10, the recipe SURVEY §0 / BASELINE.md ask for)."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    src = "measured"
    try:
        m = json.load(open(p))
        hbm, bf16 = float(m["hbm_gbs"]), float(m["bf16_tflops"])
    except Exception:
        hbm, bf16, src = 6650.0, 1590.0, "fallback"
    tf32, tf32_src = bf16 * 1.1 / 2.25, "bf16 x 1.1/2.25 nominal"
    if measure_tf32:
        try:
            tf32, tf32_src = measure_tf32_tflops(device), "measured here: cuBLAS fp32 8192^3 matmul, allow_tf32, best of 10"
        except Exception as e:  # noqa: BLE001
            tf32_src += f" (measurement failed: {e})"
    return {"hbm_gbs": hbm, "bf16_tflops": bf16, "tf32_tflops": tf32, "source": src, "tf32_source": tf32_src}


def measure_tf32_tflops(device=None, n: int = 8192, reps: int = 10) -> float:
    import torch
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        a = torch.randn(n, n, device=device)
        b = torch.randn(n, n, device=device)
        c = a @ b
        torch.cuda.synchronize(device)
        best = float("inf")
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b, out=c)
            e1.record()
            torch.cuda.synchronize(device)
            best = min(best, e0.elapsed_time(e1))
        return 2.0 * n ** 3 / (best * 1e-3) / 1e12
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


class ClockSampler:
    """nvidia-smi clocks + throttle reasons DURING the timed region (B200_PROFILING.md)."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = f"/tmp/ios_clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
        except Exception:
            rows = []
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = sorted(float(r[0]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if len(r) > 3 + i and r[3 + i].strip() == "Active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(rows[0][1]), "reasons": reasons,
                "samples": len(rows)}


def stage_roofline(g, net, q, peaks, times_ms=None):
    """Per-stage roofline: T_roof = max(F / P_tc, B / BW_HBM) with F = unpadded conv
    FLOPs and B = distinct input bytes + weight bytes + output bytes (elided concat = 0). `ms` is the
    stage's in-run attributable time when `times_ms` is given (ios_run_timeline), else the
    profiler's latency stored with the schedule."""
    from workloads.netspec import NetSpec  # noqa: F401
    esz = 2 if net.math == "bf16" else 4
    ptc = (peaks["bf16_tflops"] if net.math == "bf16" else peaks["tf32_tflops"]) * 1e12
    bw = peaks["hbm_gbs"] * 1e9
    shapes = {i: g.op_shape(i) for i in range(net.n_ops + 1)}
    rows = []
    for si, (ops, t, lat) in enumerate(q.stages):
        if times_ms is not None:
            lat = times_ms[si]
        f = 0
        wbytes = 0
        in_ids = set()
        out_b = 0
        for v in ops:
            o = net.op(v)
            n, co, ho, wo = shapes[v]
            if o.kind == "conv":
                cin = shapes[o.inputs[0]][1]
                f += 2 * n * ho * wo * co * cin * o.kh * o.kw
                wbytes += co * cin * o.kh * o.kw * esz
            elif o.kind == "sepconv":
                c = shapes[o.inputs[0]][1]
                f += 2 * n * ho * wo * c * (o.kh * o.kw + co)
                wbytes += (c * o.kh * o.kw + co * c) * esz
            elif o.kind == "linear":
                cin = shapes[o.inputs[0]][1]
                f += 2 * n * co * cin
                wbytes += co * cin * esz
            if o.kind != "concat" and o.kind != "identity":
                out_b += n * co * ho * wo * esz
                for u in o.inputs:
                    if u not in ops:
                        in_ids.add(u)
        in_b = sum(shapes[u][0] * shapes[u][1] * shapes[u][2] * shapes[u][3] * esz for u in in_ids)
        b = in_b + wbytes + out_b
        t_roof = max(f / ptc, b / bw) * 1e3
        rows.append({"ops": ops, "strategy": t, "ms": lat, "flops": f, "bytes": b, "roof_ms": t_roof,
                     "bound": "tensor" if f / ptc >= b / bw else "hbm"})
    return rows


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import workloads as W
    from paper_2011_01302_b200 import Graph

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    spec = NETS[args.net]
    # batch sharding: contiguous per-rank slices, each rank its own graph + DP schedule,
    # no collective on the hot path. Default global batch: 1 on one GPU (the BASELINE metric), 8 per
    # GPU when N > 1 (north star: partitioning only by batch, at batch >= 8; weak scaling)
    from paper_2011_01302_b200.shard import shard_range
    batch = args.batch if args.batch > 0 else (1 if world == 1 else 8 * world)
    if batch < world:
        raise SystemExit(f"global batch {batch} < {world} GPUs: batch 1 does not shard (DESIGN.md §8)")
    b0, b1 = shard_range(batch, world, rank)
    local_batch = b1 - b0
    parallelism = ("single GPU" if world == 1 else
                   f"batch-sharded {batch} over {world} GPUs ({local_batch}/rank), no collective on the hot path")
    net = W.build(args.net, math=spec["math"], batch=local_batch)
    peaks = _peaks(measure_tf32=True, device=dev)

    g = Graph.from_netspec(net, spec["math"], local)
    t0 = time.time()
    if args.latency_cache and os.path.exists(args.latency_cache):
        g.load_latency_cache(args.latency_cache)              # resume: measured stage latencies
    if args.latency_cache:
        g.autosave_latency_cache(args.latency_cache)          # checkpoint after every searched block
    q_dp = g.schedule_dp(args.r, args.s)                       # device-measured stage costs (Alg. 1)
    if args.latency_cache and not os.path.exists(args.latency_cache):
        g.save_latency_cache(args.latency_cache)
    search_s = time.time() - t0
    refine_s = 0.0
    q_ios = q_dp
    if args.refine:
        # DP optima under a family of cost models, chosen per block by in-context measurement
        # (ios_schedule_refine, DESIGN.md §6 "Measured refinement")
        t1 = time.time()
        q_ios = g.schedule_refine(args.r, args.s, reps=20, beta_us=1.0)
        refine_s = time.time() - t1
    q_seq = g.schedule_sequential()
    q_greedy = g.schedule_greedy()
    tune_s = 0.0
    if args.tune:
        # per-stage tiling variant by measurement, for every schedule alike (same kernels)
        t1 = time.time()
        for q in (q_ios, q_dp, q_seq, q_greedy):
            g.tune(q)
        tune_s = time.time() - t1
    if args.save_schedule and rank == 0:
        # exactly what is timed below, for tools/ncu_run.py --schedule (profiler replay)
        json.dump({"net": args.net, "batch": local_batch, "math": spec["math"],
                   "stages": [[ops, t] for ops, t, _ in q_ios.stages]}, open(args.save_schedule, "w"))
        g.save_tile_variants(args.save_schedule + ".variants")

    x = torch.from_numpy(net.make_input()).to(dev)
    out = torch.empty(g.output_shape(), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(int(2 * torch.cuda.get_device_properties(dev).L2_cache_size) // 4 + 1024,
                        dtype=torch.float32, device=dev)

    def timed(q, steps, warmup):
        for _ in range(warmup):
            g.run(q, x, out)
        g.sync()
        if world > 1:
            dist.barrier()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        torch.cuda.synchronize(dev)
        for i in range(steps):
            flush.fill_(float(i))                              # L2 flush between timed steps (untimed)
            evs[i][0].record(stream)
            g.run(q, x, out)
            evs[i][1].record(stream)
        torch.cuda.synchronize(dev)
        g.sync()                                               # IOS_ERR_KERNEL if any in-kernel wait timed out
        tot = sum(a.elapsed_time(b) for a, b in evs)
        t = torch.tensor([tot / steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    with ClockSampler(local) as clk:
        ms_ios = timed(q_ios, args.steps, args.warmup)
    ms_dp = timed(q_dp, max(20, args.steps // 4), args.warmup) if q_dp is not q_ios else ms_ios
    ms_seq = timed(q_seq, max(20, args.steps // 4), args.warmup)
    ms_greedy = timed(q_greedy, max(20, args.steps // 4), args.warmup)

    # end to end through the public C-ABI with HOST buffers (ios_run_host: pinned input copied in,
    # run, output copied back, synchronised), L2 flushed before every step like the timed loop;
    # host wall clock around the call (it is synchronous)
    xh_t = torch.from_numpy(net.make_input()).pin_memory()
    xh = xh_t.numpy()
    e2e_steps = max(20, args.steps // 4)
    for _ in range(args.warmup):
        yh = g.run_host(q_ios, xh)
    e2e_tot = 0.0
    for i in range(e2e_steps):
        flush.fill_(float(i))
        torch.cuda.synchronize(dev)
        t_a = time.perf_counter()
        yh = g.run_host(q_ios, xh)
        e2e_tot += time.perf_counter() - t_a
    e2e_ms = torch.tensor([e2e_tot * 1e3 / e2e_steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)

    # per-stage roofline of the IOS schedule from IN-RUN stage times: the same CUDA graph with PDL,
    # L2 flushed before each run, every stage launch stamping its span on the global timer
    # (ios_run_timeline); attributable time = end - previous stage's end
    tl = g.run_timeline(q_ios, x, out, reps=20, l2_flush=True)
    rows = stage_roofline(g, net, q_ios, peaks, times_ms=[a * 1e-3 for _, _, a in tl])
    launches_per_run = q_ios.launches()
    if rank == 0:
        tot_roof = sum(r["roof_ms"] for r in rows)
        tot_ms = sum(r["ms"] for r in rows if r["ms"] > 0)
        conv_rows = [r for r in rows if r["roof_ms"] >= 0.002 and r["flops"] > 0]
        f_tot = sum(r["flops"] for r in rows)
        b_tot = sum(r["bytes"] for r in rows)
        ptc = peaks["bf16_tflops"] if net.math == "bf16" else peaks["tf32_tflops"]
        tc_time = f_tot / (ptc * 1e9)
        hbm_time = b_tot / (peaks["hbm_gbs"] * 1e6)
        bound = "tensor" if tc_time >= hbm_time else "hbm"
        if bound == "tensor":
            achieved, peak, unit = f_tot / (tot_ms * 1e9), ptc, "TFLOP/s"
        else:
            achieved, peak, unit = b_tot / (tot_ms * 1e6), peaks["hbm_gbs"], "GB/s"
        cpu = cpu_baseline(net, args.cpu_sample_s)
        traffic = None
        tp = os.path.join(ROOT, "profiles", f"traffic_{args.net}.json")
        if os.path.exists(tp) and local_batch == 1:
            try:
                traffic = json.load(open(tp)).get("bytes_per_step")
            except Exception:
                traffic = None
        line = {
            "metric": METRIC,
            "value": round(ms_ios, 4),
            "unit": "ms",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_ios, 4),
            "higher_is_better": False,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "bf16" if net.math == "bf16" else "tf32",
            "data": "synthetic (seeded N(0,1) input, He-init weights, DESIGN.md input recipe)",
            "config": {"workload": spec["desc"] if batch == 1 else spec["desc"].replace("batch 1", f"batch {batch}"),
                       "net": args.net, "batch": batch, "schedule": f"IOS-Both r={args.r} s={args.s}" + (" + measured refinement" if args.refine else ""),
                       "parallelism": parallelism, "l2": "flushed before every timed step",
                       "stages": len(q_ios.stages), "launches_per_run": launches_per_run},
            "ios_dp_ms": round(ms_dp, 4),
            "sequential_ms": round(ms_seq, 4),
            "greedy_ms": round(ms_greedy, 4),
            "speedup_vs_sequential": round(ms_seq / ms_ios, 3),
            "speedup_vs_greedy": round(ms_greedy / ms_ios, 3),
            "images_per_s": round(batch * 1000.0 / ms_ios, 1),
            "search_s": round(search_s, 2),
            "refine_s": round(refine_s, 2),
            "refine_stats": {"candidates": q_ios.stats[3] // 1000, "blocks_not_from_plain_dp": q_ios.stats[3] % 1000}
            if args.refine else None,
            "tune_s": round(tune_s, 2),
            "search_stats": {"states": q_dp.stats[0], "transitions": q_dp.stats[1], "stages_measured": q_dp.stats[2]},
            "roofline": {"bound": bound, "achieved": round(achieved, 2), "peak": round(peak, 1), "unit": unit,
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "peak_source": peaks["source"] + ("" if net.math == "bf16" else "; tf32: " + peaks["tf32_source"]),
                         "kernel": "ios_stage_kernel (all stage launches of one inference; algorithmic bytes or FLOPs of "
                                   "the schedule / sum of in-run stage times, ios_run_timeline, L2 flushed per run)"},
            "stage_roofline": {"frac_sum": round(tot_roof / tot_ms, 4) if tot_ms else None,
                               "conv_stages": len(conv_rows),
                               "conv_stages_ge_50pct": sum(1 for r in conv_rows if r["ms"] > 0 and r["roof_ms"] / r["ms"] >= 0.5),
                               "best_stage_frac": round(max((r["roof_ms"] / r["ms"] for r in rows if r["ms"] > 0), default=0), 4),
                               "roof_ms_sum": round(tot_roof, 4), "stage_ms_sum_in_run": round(tot_ms, 4),
                               "tf32_peak_tflops": round(peaks["tf32_tflops"], 1)},
            "cpu_baseline": cpu,
            "e2e": {"value": round(float(e2e_ms.item()), 4), "unit": "ms",
                    "h2d_bytes_per_step": int(xh_t.numel() * 4), "d2h_bytes_per_step": int(np.prod(g.output_shape()) * 4),
                    "how": "ios_run_host (C-ABI, pinned host buffers), host wall clock, L2 flushed before each step"},
            "gpu_launches": int(launches_per_run * args.steps),
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _oracle_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(net, budget_s: float):
    """The oracle as it stands (plain NumPy float64 sequential executor), timed on this host with the
    BLAS thread pool sized to the affinity cores (its convolutions are single-threaded einsums; its
    matmuls use the pool)."""
    from oracle import OracleGraph
    threads = _oracle_threads()
    try:
        from threadpoolctl import threadpool_limits
        ctx = threadpool_limits(limits=threads)
    except Exception:
        ctx = None
    og = OracleGraph(net)
    x = net.make_input()
    times = []
    t_start = time.time()
    while not times or (time.time() - t_start < budget_s and len(times) < 3):
        t0 = time.perf_counter()
        og.run_sequential(x)
        times.append(time.perf_counter() - t0)
    if ctx is not None and hasattr(ctx, "unregister"):
        ctx.unregister()
    ms = sorted(times)[len(times) // 2] * 1e3
    return {"value": round(ms, 2), "unit": "ms", "cores": threads, "kind": "oracle",
            "sample": f"{len(times)} full inference(s) of the same network, batch {net.input_shape[0]} "
                      f"(run_sequential, float64; BLAS threads = {threads}, conv einsums single-threaded)"}


def run_reference(args):
    """--impl reference: the CPU oracle timed as it stands (the tier's reference arm)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import workloads as W
    from oracle import OracleGraph
    spec = NETS[args.net]
    net = W.build(args.net, math=spec["math"])
    threads = _oracle_threads()
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(limits=threads)
    except Exception:
        pass
    og = OracleGraph(net)
    x = net.make_input()
    for _ in range(min(args.warmup, 1)):
        og.run_sequential(x)
    steps = max(1, min(args.steps, 3))
    t0 = time.perf_counter()
    for _ in range(steps):
        og.run_sequential(x)
    ms = (time.perf_counter() - t0) * 1e3 / steps
    line = {"impl": "reference", "metric": METRIC, "value": round(ms, 2), "unit": "ms", "n_gpus": world,
            "steps": steps, "warmup": min(args.warmup, 1), "ms_per_step": round(ms, 2), "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": spec["desc"], "net": args.net, "batch": 1, "schedule": "sequential (oracle)"},
            "cpu_baseline": {"value": round(ms, 2), "unit": "ms", "cores": threads, "kind": "oracle",
                             "sample": f"{steps} full batch-1 inference(s), float64 NumPy (BLAS threads = {threads})"},
            "e2e": {"value": round(ms, 2), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def _relaunch_distributed(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: re-exec under torch.distributed.run, one rank per GPU."""
    import random
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(random.randint(20000, 40000)),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--net", default="inception_v3", choices=sorted(NETS))
    ap.add_argument("--batch", type=int, default=0,
                    help="global batch, sharded across the ranks (default: 1 on one GPU, 8 per GPU when N > 1)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--r", type=int, default=3)
    ap.add_argument("--s", type=int, default=8)
    ap.add_argument("--cpu-sample-s", type=float, default=10.0)
    ap.add_argument("--latency-cache", default="", help="load (if present) / save the DP's stage-latency cache")
    ap.add_argument("--tune", type=int, default=1, help="1: ios_schedule_tune every schedule (per-stage tiling), 0: default tiling")
    ap.add_argument("--refine", type=int, default=1, help="1: ios_schedule_refine (DP candidates chosen per block in context)")
    ap.add_argument("--save-schedule", default="", help="write the timed IOS schedule (+ .variants) for tools/ncu_run.py")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_relaunch_distributed(args.gpus))
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}; using WORLD_SIZE", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
