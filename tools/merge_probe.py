"""Concurrent vs merged latency of mergeable stages (verdict r1 #6 / P:566-571 merge flip):
  python tools/merge_probe.py --net inception_v3 --batch 1 --stages "8,9,11;97,98,101;99,100;103,104" """
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa
import workloads as W  # noqa
from bench import NETS  # noqa
from paper_2011_01302_b200 import Graph, MERGE, CONCURRENT  # noqa
ap = argparse.ArgumentParser()
ap.add_argument("--net", default="inception_v3")
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--stages", default="8,9,11;97,98,101;99,100;103,104")
a = ap.parse_args()
net = W.build(a.net, math=NETS[a.net]["math"], batch=a.batch)
g = Graph.from_netspec(net, NETS[a.net]["math"])
x = torch.from_numpy(net.make_input()).cuda()
g.run(g.schedule_sequential(), x)
g.sync()
for st in a.stages.split(";"):
    ops = [int(v) for v in st.split(",")]
    names = ",".join(net.op(v).name.split(".")[-1] for v in ops)
    c = g.stage_latency(ops, CONCURRENT, trials=5, reps=20) * 1e3
    m = g.stage_latency(ops, MERGE, trials=5, reps=20) * 1e3
    print(f"batch {a.batch} [{names}] concurrent {c:.2f} us merge {m:.2f} us -> {'MERGE' if m <= c else 'concurrent'}", flush=True)
