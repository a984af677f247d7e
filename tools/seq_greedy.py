"""Sequential / greedy schedule latency of a network (no DP search): quick A/B of kernel knobs in
the real launch path (CUDA graph, PDL, L2 flushed before each timed step).

  IOS_FUSE_DW=0 python tools/seq_greedy.py --net nasnet_a_large
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
ap.add_argument("--net", default="nasnet_a_large")
ap.add_argument("--steps", type=int, default=30)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--tune", type=int, default=0, help="1: stage-tune both schedules first (ios_schedule_tune)")
a = ap.parse_args()
math = NETS[a.net]["math"]
net = W.build(a.net, math=math, batch=a.batch)
g = Graph.from_netspec(net, math)
x = torch.from_numpy(net.make_input()).cuda()
out = torch.empty(g.output_shape(), dtype=torch.float32, device="cuda")
flush = torch.empty(int(2 * torch.cuda.get_device_properties(0).L2_cache_size) // 4 + 1024, device="cuda")
res = {}
for name, q in (("sequential", g.schedule_sequential()), ("greedy", g.schedule_greedy())):
    if a.tune:
        g.tune(q)
    for _ in range(3):
        g.run(q, x, out)
    torch.cuda.synchronize()
    tot = 0.0
    for i in range(a.steps):
        flush.fill_(float(i))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.run(q, x, out)
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    res[name] = round(tot / a.steps, 4)
print(a.net, res)
