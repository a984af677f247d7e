"""Per-op (sequential-schedule) stage latencies vs roofline, for kernel tuning."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W
from paper_2011_01302_b200 import Graph
from bench import stage_roofline, _peaks
name = sys.argv[1] if len(sys.argv) > 1 else "inception_v3"
net = W.build(name)
g = Graph.from_netspec(net)
q = g.schedule_sequential()
rows = []
for i in range(1, net.n_ops + 1):
    ms = g.stage_latency([i])
    rows.append(ms)
qq = g.schedule([([i], 0) for i in range(1, net.n_ops + 1)])
peaks = _peaks()
rr = stage_roofline(g, net, q, peaks)
tot = 0
for i, (ms, r) in enumerate(zip(rows, rr), start=1):
    o = net.op(i)
    tot += ms
    print(f"{i:4d} {o.kind:8s} {o.name[:28]:28s} {str(g.op_shape(i)):22s} ms={ms*1e3:8.1f}us roof={r['roof_ms']*1e3:7.2f}us {r['bound']}")
print("total", tot)
