"""N2: batch-specialised schedules, Table 3 / Fig. 9 of the paper.

For every batch b the DP searches Inception V3 at that batch (device-measured stage costs); then
every schedule is run at every batch (the schedules are op-id stage lists, valid at any batch) and
timed end to end. Also reports whether the 1x3/3x1 pair of Mixed_7b/7c is merged at each batch
(the paper's merge flip at large batch).

  python tools/batch_specialise.py --batches 1 16 32 64 128 --out profiles/r1_batch_specialise.json
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2011_01302_b200 import Graph, MERGE  # noqa: E402


def time_ms(g, q, x, out, iters, reps=5):
    st = torch.cuda.current_stream()
    for _ in range(3):
        g.run(q, x, out)
    torch.cuda.synchronize()
    res = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(iters):
            g.run(q, x, out)
        b.record(st)
        torch.cuda.synchronize()
        res.append(a.elapsed_time(b) / iters)
    res.sort()
    return res[len(res) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="inception_v3")
    ap.add_argument("--math", default="tf32")
    ap.add_argument("--batches", type=int, nargs="+", default=[1, 16, 32, 64, 128])
    ap.add_argument("--cache-dir", default="gpurun_out")
    ap.add_argument("--out", default="gpurun_out/batch_specialise.json")
    a = ap.parse_args()
    graphs, nets, scheds, info = {}, {}, {}, {}
    for b in a.batches:
        net = W.build(a.net, math=a.math, batch=b)
        g = Graph.from_netspec(net, a.math)
        lc = os.path.join(a.cache_dir, f"lc_{a.net}_b{b}.txt")
        if os.path.exists(lc):
            g.load_latency_cache(lc)
        g.autosave_latency_cache(lc)
        t0 = time.time()
        q = g.schedule_dp(3, 8)
        info[b] = {"search_s": round(time.time() - t0, 1), "dp_cost_ms": q.cost,
                   "stats": list(q.stats), "n_stages": len(q.stages)}
        scheds[b] = [(list(ops), int(t)) for ops, t, _ in q.stages]
        graphs[b], nets[b] = g, net
        # the Mixed_7b/7c 1x3 / 3x1 pairs: merged at this batch?
        pairs = []
        for tag in ("Mixed_7b", "Mixed_7c"):
            for br in ("b3x3", "b3x3dbl"):
                ids = [i for i in range(1, net.n_ops + 1) if net.op(i).name in (f"{tag}.{br}_2a", f"{tag}.{br}_3a",
                                                                                  f"{tag}.{br}_2b", f"{tag}.{br}_3b")]
                if len(ids) == 2:
                    st = [t for ops, t in scheds[b] if ids[0] in ops and ids[1] in ops]
                    pairs.append({"pair": f"{tag}.{br}", "ops": ids, "same_stage": bool(st),
                                  "merged": bool(st and st[0] == MERGE)})
        info[b]["pairs_1x3_3x1"] = pairs
        print(f"batch {b}: search {info[b]['search_s']}s, {len(q.stages)} stages, dp cost {q.cost:.4f} ms, "
              f"merged pairs {[p['pair'] for p in pairs if p['merged']]}", flush=True)
    table = {}
    for bj in a.batches:
        g, net = graphs[bj], nets[bj]
        x = torch.from_numpy(net.make_input()).cuda()
        out = torch.empty(g.output_shape(), dtype=torch.float32, device="cuda")
        iters = max(3, 40 // bj)
        row = {}
        for bi in a.batches:
            row[f"sched_b{bi}"] = time_ms(g, g.schedule(scheds[bi]), x, out, iters)
        row["sequential"] = time_ms(g, g.schedule_sequential(), x, out, iters)
        row["greedy"] = time_ms(g, g.schedule_greedy(), x, out, iters)
        table[f"run_b{bj}"] = row
        print(f"run at batch {bj}: " + " ".join(f"{k}={v:.3f}" for k, v in row.items()), flush=True)
    json.dump({"net": a.net, "math": a.math, "batches": a.batches, "search": {str(k): v for k, v in info.items()},
               "latency_ms": table, "schedules": {str(k): v for k, v in scheds.items()}}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
