"""ios_stage_latency of given stages (e.g. A/B of kernel knobs on one stage):
  python tools/stage_latency.py --net inception_v3 --stages "1,2,3;5,6,7" """
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa
import workloads as W  # noqa
from bench import NETS  # noqa
from paper_2011_01302_b200 import Graph  # noqa
ap = argparse.ArgumentParser()
ap.add_argument("--net", default="inception_v3")
ap.add_argument("--stages", default="1,2,3;5,6,7")
a = ap.parse_args()
net = W.build(a.net, math=NETS[a.net]["math"])
g = Graph.from_netspec(net, NETS[a.net]["math"])
x = torch.from_numpy(net.make_input()).cuda()
g.run(g.schedule_sequential(), x)
g.sync()
out = []
for st in a.stages.split(";"):
    ops = [int(v) for v in st.split(",")]
    out.append(f"[{st}]:{g.stage_latency(ops, 0, trials=5, reps=20) * 1e3:.2f}")
print(" ".join(out))
