"""One IOS-scheduled inference bracketed by cudaProfilerStart/Stop, for
`ncu --profile-from-start off` launch lists / DRAM traffic of exactly one step.

  ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,\
dram__bytes_write.sum --csv --log-file out.csv python tools/ncu_run.py --net inception_v3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from bench import NETS  # noqa: E402
from paper_2011_01302_b200 import Graph  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--net", default="inception_v3")
ap.add_argument("--latency-cache", default="")
ap.add_argument("--schedule", default="", help="replay the schedule + tile variants bench.py --save-schedule wrote")
a = ap.parse_args()
if a.schedule:
    import json
    sj = json.load(open(a.schedule))
    a.net = sj["net"]
math = NETS[a.net]["math"]
net = W.build(a.net, math=math, batch=sj["batch"]) if a.schedule else W.build(a.net, math=math)
g = Graph.from_netspec(net, math)
if a.schedule:
    # exactly the stages and tiling variants the bench timed
    q = g.schedule([(ops, t) for ops, t in sj["stages"]])
    g.load_tile_variants(a.schedule + ".variants")
else:
    if a.latency_cache and os.path.exists(a.latency_cache):
        g.load_latency_cache(a.latency_cache)
    q = g.schedule_dp(3, 8)
x = torch.from_numpy(net.make_input()).cuda()
out = torch.empty(g.output_shape(), dtype=torch.float32, device="cuda")
for _ in range(3):
    g.run(q, x, out)
torch.cuda.synchronize()
flush = torch.empty(int(2 * torch.cuda.get_device_properties(0).L2_cache_size) // 4, device="cuda")
flush.fill_(1.0)
torch.cuda.synchronize()
torch.cuda.profiler.start()
g.run(q, x, out)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("stages", len(q.stages), "launches", q.launches())
