"""Single-op stages of a network, each launched once between cudaProfilerStart/Stop (for
`ncu --profile-from-start off --set full`):  python tools/ncu_ops.py --net squeezenet --batch 128 --ops 1,5,38"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa
import workloads as W  # noqa
from bench import NETS  # noqa
from paper_2011_01302_b200 import Graph  # noqa
ap = argparse.ArgumentParser()
ap.add_argument("--net", default="squeezenet")
ap.add_argument("--batch", type=int, default=128)
ap.add_argument("--ops", default="1,5,38")
a = ap.parse_args()
net = W.build(a.net, math=NETS[a.net]["math"], batch=a.batch)
g = Graph.from_netspec(net, NETS[a.net]["math"])
x = torch.from_numpy(net.make_input()).cuda()
ops = [int(v) for v in a.ops.split(",")]
q = g.schedule([([i], 0) for i in range(1, net.n_ops + 1)])
g.run(q, x)
g.sync()
for v in ops:
    g.stage_latency([v], 0, warmup=2, trials=1, reps=1)   # builds/warms the plan
torch.cuda.synchronize()
torch.cuda.profiler.start()
for v in ops:
    g.stage_latency([v], 0, warmup=1, trials=1, reps=1)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
