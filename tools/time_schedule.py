"""Time one saved schedule (bench.py --save-schedule JSON) through ios_run: CUDA graph + PDL,
L2 flushed before every timed step. For A/B runs of kernel / tiling knobs on the exact stages the
bench timed (tools/_abenv.sh style).

  python tools/time_schedule.py profiles/r2_sched_inception.json [--tune 1] [--steps 50]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2011_01302_b200 import Graph  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("schedule")
ap.add_argument("--tune", type=int, default=1)
ap.add_argument("--steps", type=int, default=50)
a = ap.parse_args()
sj = json.load(open(a.schedule))
net = W.build(sj["net"], math=sj["math"], batch=sj["batch"])
g = Graph.from_netspec(net, sj["math"])
q = g.schedule([(o, t) for o, t in sj["stages"]])
if a.tune:
    g.tune(q)
x = torch.from_numpy(net.make_input()).cuda()
out = torch.empty(g.output_shape(), dtype=torch.float32, device="cuda")
flush = torch.empty(int(2 * torch.cuda.get_device_properties(0).L2_cache_size) // 4 + 1024, device="cuda")
for _ in range(5):
    g.run(q, x, out)
g.sync()
tot = 0.0
for i in range(a.steps):
    flush.fill_(float(i))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.run(q, x, out)
    e1.record()
    torch.cuda.synchronize()
    tot += e0.elapsed_time(e1)
g.sync()
print(sj["net"], os.path.basename(a.schedule), "tuned" if a.tune else "untuned", round(tot / a.steps, 4), "ms")
