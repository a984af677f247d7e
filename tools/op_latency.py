"""Single-op stage latencies (ios_stage_latency) of selected ops, e.g. for split-K sweeps:
  IOS_MAX_SPLIT=1 python tools/op_latency.py --net inception_v3 --ops 10,42,99"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa
import workloads as W  # noqa
from bench import NETS  # noqa
from paper_2011_01302_b200 import Graph  # noqa
ap = argparse.ArgumentParser()
ap.add_argument("--net", default="inception_v3")
ap.add_argument("--ops", default="10,13,42,99")
a = ap.parse_args()
net = W.build(a.net, math=NETS[a.net]["math"])
g = Graph.from_netspec(net, NETS[a.net]["math"])
x = torch.from_numpy(net.make_input()).cuda()
g.run(g.schedule_sequential(), x)
g.sync()
res = []
for v in (int(t) for t in a.ops.split(",")):
    res.append(f"{v}:{g.stage_latency([v], 0, trials=5, reps=20) * 1e3:.2f}")
print(" ".join(res))
