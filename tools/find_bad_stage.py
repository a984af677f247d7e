"""Measure every (3, 8)-pruned candidate stage of a network in DP order; report the first failure."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W
from oracle import OracleGraph, scheduler as S
from paper_2011_01302_b200 import Graph, MERGE
name = sys.argv[1] if len(sys.argv) > 1 else "inception_v3"
net = W.build(name)
og = OracleGraph(net)
g = Graph.from_netspec(net)
seen = set()
for b in og.block_ids:
    mem = og.block_members[b]
    full = (1 << len(mem)) - 1
    # all states reachable: BFS
    states = [full]; vis = {full}
    while states:
        st = states.pop()
        for sp in S.endings(og.succ[b], og.pred[b], st, 3, 8):
            ops = og.block_mask_ops(b, sp)
            for t in ([0, 1] if og.mergeable(ops) else [0]):
                key = (tuple(ops), t)
                if key in seen: continue
                seen.add(key)
                try:
                    g.stage_latency(ops, t, warmup=1, trials=1, reps=1)
                except Exception as e:
                    print("FAIL", ops, t, [net.op(v).name for v in ops], e, flush=True)
                    sys.exit(1)
            nxt = st & ~sp
            if nxt and nxt not in vis:
                vis.add(nxt); states.append(nxt)
print("all ok", len(seen))
