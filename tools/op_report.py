"""Per-op single-stage latency vs roofline (where does the sequential time go?).

  python tools/op_report.py --net nasnet_a_large [--ops 1-60] [--top 30]
"""
import argparse
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from bench import NETS, stage_roofline, _peaks  # noqa: E402
from paper_2011_01302_b200 import Graph  # noqa: E402


class _Q:
    def __init__(self, stages):
        self.stages = stages


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="nasnet_a_large")
    ap.add_argument("--ops", default="")
    ap.add_argument("--top", type=int, default=30)
    a = ap.parse_args()
    math = NETS[a.net]["math"] if a.net in NETS else "tf32"
    net = W.build(a.net, math=math)
    g = Graph.from_netspec(net, math)
    if a.ops:
        lo, hi = (int(v) for v in a.ops.split("-"))
        ids = list(range(lo, hi + 1))
    else:
        ids = list(range(1, net.n_ops + 1))
    stages = []
    for v in ids:
        if net.op(v).kind in ("concat", "identity"):
            continue
        stages.append(([v], 0, g.stage_latency([v], 0, warmup=3, trials=3, reps=10)))
    rows = stage_roofline(g, net, _Q(stages), _peaks())
    by_kind = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for r in rows:
        o = net.op(r["ops"][0])
        k = o.kind + (f"{o.kh}x{o.kw}s{o.sh}" if o.kind in ("conv", "sepconv") else "") + \
            ("+relu_pre" if getattr(o, "relu_pre", False) and o.kind == "conv" else "")
        by_kind[k][0] += 1
        by_kind[k][1] += r["ms"]
        by_kind[k][2] += r["roof_ms"]
    print(f"{'kind':28s} {'n':>4s} {'sum us':>9s} {'roof us':>8s}")
    for k, (n, ms, roof) in sorted(by_kind.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:28s} {n:4d} {ms*1e3:9.1f} {roof*1e3:8.2f}")
    print("worst ops (ms - roof):")
    for r in sorted(rows, key=lambda r: r["roof_ms"] - r["ms"])[:a.top]:
        v = r["ops"][0]
        o = net.op(v)
        shp = g.op_shape(v)
        ishp = g.op_shape(o.inputs[0])
        print(f"  op {v:4d} {o.kind:8s} {o.name[:28]:28s} in={ishp} out={shp} k={o.kh}x{o.kw}s{o.sh} "
              f"{r['ms']*1e3:8.1f}us roof {r['roof_ms']*1e3:6.2f}us")


if __name__ == "__main__":
    main()
