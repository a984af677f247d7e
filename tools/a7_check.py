"""Stage profiler (ios_stage_latency, the DP's cost) vs in-run stage times (ios_run_timeline):
per stage of a schedule, profiled ms vs attributable in-run time (warm L2 and L2 flushed per run).

  python tools/a7_check.py --net inception_v3 [--schedule ios|seq|greedy]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from bench import NETS, _peaks, stage_roofline  # noqa: E402
from paper_2011_01302_b200 import Graph  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--net", default="inception_v3")
ap.add_argument("--schedule", default="ios")
ap.add_argument("--tune", type=int, default=1)
ap.add_argument("--batch", type=int, default=1)
a = ap.parse_args()
math = NETS[a.net]["math"]
net = W.build(a.net, math=math, batch=a.batch)
g = Graph.from_netspec(net, math)
q = {"ios": lambda: g.schedule_dp(3, 8), "seq": g.schedule_sequential, "greedy": g.schedule_greedy}[a.schedule]()
if a.tune:
    g.tune(q)
x = torch.from_numpy(net.make_input()).cuda()
out = g.run(q, x)
g.sync()
warm = g.run_timeline(q, x, out, reps=20, l2_flush=False)
cold = g.run_timeline(q, x, out, reps=20, l2_flush=True)
prof = [g.stage_latency(ops, t) * 1e3 if ops and net.op(ops[0]).kind != "concat" or len(ops) > 1 else 0.0
        for ops, t, _ in q.stages]
rows = stage_roofline(g, net, q, _peaks(), times_ms=[c[2] * 1e-3 for c in cold])
print(f"{'i':>3s} {'prof':>7s} {'warm':>7s} {'cold':>7s} {'span':>7s} {'roof':>6s}  ops")
for i, ((ops, t, _), p, w, c, r) in enumerate(zip(q.stages, prof, warm, cold, rows)):
    print(f"{i:3d} {p:7.2f} {w[2]:7.2f} {c[2]:7.2f} {c[1]-c[0]:7.2f} {r['roof_ms']*1e3:6.2f} {r['bound']:6s} "
          f"F={r['flops']/1e9:6.2f}G B={r['bytes']/1e6:7.1f}MB  {ops} {[net.op(v).name for v in ops][:3]}")
P, Wm, Cd = sum(prof), sum(w[2] for w in warm), sum(c[2] for c in cold)
print(f"sum: profiled {P:.1f} us, in-run warm {Wm:.1f} us, in-run L2-flushed {Cd:.1f} us, roof {sum(r['roof_ms'] for r in rows)*1e3:.1f} us")
nz = [(p, c[2]) for p, c in zip(prof, cold) if p > 0]
ratio = np.array([c / p for p, c in nz])
print(f"in-run(cold)/profiled per stage: median {np.median(ratio):.2f} min {ratio.min():.2f} max {ratio.max():.2f}")
