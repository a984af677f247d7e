"""Print the IOS schedule of a network (per stage: ops, strategy, measured ms, roofline ms)."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W
from paper_2011_01302_b200 import Graph
from bench import NETS, stage_roofline, _peaks
ap = argparse.ArgumentParser()
ap.add_argument("--net", default="inception_v3")
ap.add_argument("--latency-cache", default="")
ap.add_argument("--json", default="")
ap.add_argument("--r", type=int, default=3)
ap.add_argument("--s", type=int, default=8)
a = ap.parse_args()
net = W.build(a.net, math=NETS[a.net]["math"])
g = Graph.from_netspec(net, NETS[a.net]["math"])
if a.latency_cache and os.path.exists(a.latency_cache):
    g.load_latency_cache(a.latency_cache)
if a.latency_cache:
    g.autosave_latency_cache(a.latency_cache)
q = g.schedule_dp(a.r, a.s)
if a.latency_cache and not os.path.exists(a.latency_cache):
    g.save_latency_cache(a.latency_cache)
rows = stage_roofline(g, net, q, _peaks())
for i, r in enumerate(rows):
    names = ",".join(net.op(v).name.split(".")[-1] for v in r["ops"])
    print(f"{i:3d} {'M' if r['strategy'] else 'C'} ms={r['ms']*1e3:7.1f}us roof={r['roof_ms']*1e3:6.2f}us {r['bound']:6s} ops={r['ops']} [{names[:80]}]")
print("sum stage ms", sum(r["ms"] for r in rows), "roof", sum(r["roof_ms"] for r in rows))
if a.json:
    json.dump(rows, open(a.json, "w"))
