"""IOS-Merge / IOS-Parallel / IOS-Both (Fig. 6) and the pruning sweep
r in {1, 2, 3} x s in {3, 8} (Fig. 10) on the device: schedule latency (ms, CUDA-graph
replay, L2 flushed) and search cost (s, stages measured) per setting.

python tools/sweep_strategies.py --net inception_v3 [--json out.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import workloads as W  # noqa: E402
from bench import NETS  # noqa: E402
from paper_2011_01302_b200 import Graph  # noqa: E402


def time_schedule(g, q, x, out, flush, steps=50, warmup=5):
    for _ in range(warmup):
        g.run(q, x, out)
    torch.cuda.synchronize()
    tot = 0.0
    for i in range(steps):
        flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.run(q, x, out)
        b.record()
        b.synchronize()
        tot += a.elapsed_time(b)
    return tot / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="inception_v3")
    ap.add_argument("--json", default="")
    ap.add_argument("--latency-cache", default="")
    a = ap.parse_args()
    spec = NETS[a.net]
    net = W.build(a.net, math=spec["math"])
    g = Graph.from_netspec(net, spec["math"])
    if a.latency_cache and os.path.exists(a.latency_cache):
        g.load_latency_cache(a.latency_cache)
    x = torch.from_numpy(net.make_input()).cuda()
    out = torch.empty(g.output_shape(), device="cuda")
    flush = torch.empty(int(2 * torch.cuda.get_device_properties(0).L2_cache_size) // 4, device="cuda")
    rows = []
    for name, q, search in [("sequential", g.schedule_sequential(), 0.0), ("greedy", g.schedule_greedy(), 0.0)]:
        rows.append({"schedule": name, "ms": time_schedule(g, q, x, out, flush), "search_s": search,
                     "stages": len(q.stages)})
    for strategies in ("both", "parallel", "merge"):
        for r, s in ([(3, 8)] if strategies != "both" else [(1, 3), (1, 8), (2, 3), (2, 8), (3, 3), (3, 8)]):
            t0 = time.time()
            q = g.schedule_dp(r, s, strategies=strategies)
            search = time.time() - t0
            n_merge = sum(1 for _, t, _ in q.stages if t == 1)
            rows.append({"schedule": f"IOS-{strategies.capitalize()}", "r": r, "s": s,
                         "ms": time_schedule(g, q, x, out, flush), "search_s": round(search, 2),
                         "stages": len(q.stages), "merge_stages": n_merge,
                         "stages_measured": q.stats[2], "transitions": q.stats[1]})
            print(json.dumps(rows[-1]), flush=True)
    if a.latency_cache and not os.path.exists(a.latency_cache):
        g.save_latency_cache(a.latency_cache)
    for r in rows:
        print(json.dumps(r))
    if a.json:
        json.dump({"net": a.net, "math": spec["math"], "rows": rows}, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
