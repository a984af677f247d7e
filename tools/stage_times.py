"""Per-stage in-run times of a saved schedule (bench.py --save-schedule): the schedule's own CUDA
graph, L2 flushed per run (ios_run_timeline), next to each stage's roofline and its dependent-GEMM
depth (the longest chain of GEMM members inside the stage: the number of dependent conv links the
stage pays for in one launch).

  python tools/stage_times.py --schedule profiles/r2_sched_inception.json
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from bench import _peaks, stage_roofline  # noqa: E402
from paper_2011_01302_b200 import Graph  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--schedule", required=True)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--variants", type=int, default=1, help="0: ignore the saved tile variants (IOS_TILE_VARIANT applies)")
a = ap.parse_args()
sj = json.load(open(a.schedule))
net = W.build(sj["net"], math=sj["math"], batch=sj["batch"])
g = Graph.from_netspec(net, sj["math"])
q = g.schedule([(ops, t) for ops, t in sj["stages"]])
if a.variants and os.path.exists(a.schedule + ".variants"):
    g.load_tile_variants(a.schedule + ".variants")
x = torch.from_numpy(net.make_input()).cuda()
out = torch.empty(g.output_shape(), dtype=torch.float32, device="cuda")
for _ in range(3):
    g.run(q, x, out)
torch.cuda.synchronize()
tl = g.run_timeline(q, x, out, reps=a.reps, l2_flush=True)
rows = stage_roofline(g, net, q, _peaks(), times_ms=[t * 1e-3 for _, _, t in tl])
gemm_kinds = ("conv", "sepconv", "linear")
tot = 0.0
tot_links = 0
for (ops, t), r, (s0, s1, att) in zip(sj["stages"], rows, tl):
    depth = {}
    for v in ops:
        o = net.op(v)
        d = max([depth.get(u, 0) for u in o.inputs if u in ops] or [0])
        depth[v] = d + (1 if o.kind in gemm_kinds else 0)
    links = max(depth.values())
    tot += att
    tot_links += links
    names = ",".join(net.op(v).name.split(".")[-1] for v in ops)
    print(f"{str(ops):34s} T={t} links={links} {att:7.1f} us (span {s1 - s0:6.1f}) roof {r['roof_ms'] * 1e3:6.2f} us "
          f"{r['bound']:6s} {names[:70]}")
print(f"total {tot:.1f} us over {len(tl)} stages, {tot_links} dependent GEMM links "
      f"({tot / max(1, tot_links):.2f} us per link)")
