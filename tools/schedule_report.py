"""Print the IOS schedule of a network (per stage: ops, strategy, measured ms, roofline ms);
--trace N also prints the per-CTA timeline (ios_stage_trace) of the N stages furthest above
their roofline."""
import argparse, ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads as W
from paper_2011_01302_b200 import Graph
from paper_2011_01302_b200.ios import lib, _check, _i32
from bench import NETS, stage_roofline, _peaks
ap = argparse.ArgumentParser()
ap.add_argument("--net", default="inception_v3")
ap.add_argument("--latency-cache", default="")
ap.add_argument("--json", default="")
ap.add_argument("--r", type=int, default=3)
ap.add_argument("--s", type=int, default=8)
ap.add_argument("--trace", type=int, default=0)
ap.add_argument("--tune", type=int, default=0)
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
if a.tune:
    g.tune(q)
rows = stage_roofline(g, net, q, _peaks())
for i, r in enumerate(rows):
    names = ",".join(net.op(v).name.split(".")[-1] for v in r["ops"])
    print(f"{i:3d} {'M' if r['strategy'] else 'C'} ms={r['ms']*1e3:7.1f}us roof={r['roof_ms']*1e3:6.2f}us {r['bound']:6s} "
          f"F={r['flops']/1e6:7.1f}M B={r['bytes']/1e6:6.2f}MB ops={r['ops']} [{names[:80]}]")
print("sum stage ms", sum(r["ms"] for r in rows), "roof", sum(r["roof_ms"] for r in rows))
if a.json:
    json.dump(rows, open(a.json, "w"))
if a.trace:
    lib.ios_stage_trace.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.c_int32, C.c_int32, C.POINTER(C.c_uint64),
                                    C.c_int32, C.POINTER(C.c_int32)]
    names = ["entry", "prologue", "A1 issued", "prod done", "mma done", "acc1 ready", "epi done", "teardown", "exit",
             "A2 issued", "A3 issued", "own prologue", "A landed", "e:13", "e:14", "e:15"]
    for r in sorted(rows, key=lambda r: r["roof_ms"] - r["ms"])[:a.trace]:
        ops, t = r["ops"], r["strategy"]
        buf = (C.c_uint64 * (148 * 16))()
        grid = C.c_int32()
        _check(lib.ios_stage_trace(g.handle, _i32(ops), len(ops), t, buf, 148 * 16, C.byref(grid)))
        arr = np.array(buf[:grid.value * 16], dtype=np.int64).reshape(grid.value, 16)
        t0 = arr[:, 0][arr[:, 0] > 0].min()
        ent = (arr[:, :1] - t0) / 1000.0      # slot 0 globaltimer ns; others SM cycles + 1 (ios.h)
        rel = np.where(arr > 0, ent + (arr - 1) / 1965.0, np.nan)
        rel[:, 0] = ent[:, 0]
        print(f"stage {ops} T={t} {r['ms']*1e3:.1f} us (roof {r['roof_ms']*1e3:.2f}), grid {grid.value}; "
              "us since first entry (min/median/max over CTAs):")
        for k, nm in enumerate(names):
            col = rel[:, k]
            col = col[~np.isnan(col)]
            if len(col):
                print(f"   {nm:11s} {col.min():8.2f} {np.median(col):8.2f} {col.max():8.2f}  (n={len(col)})")
