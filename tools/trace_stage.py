"""Per-CTA timeline of one stage launch (ios_stage_trace), relative to the earliest CTA entry."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads as W
from paper_2011_01302_b200 import Graph
from paper_2011_01302_b200.ios import lib, _check, _i32
net = W.build(sys.argv[1])
g = Graph.from_netspec(net)
stages = eval(sys.argv[2])
lib.ios_stage_trace.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.c_int32, C.c_int32, C.POINTER(C.c_uint64), C.c_int32, C.POINTER(C.c_int32)]
for ops, t in stages:
    ms = g.stage_latency(ops, t)
    buf = (C.c_uint64 * (148 * 16))()
    grid = C.c_int32()
    _check(lib.ios_stage_trace(g.handle, _i32(ops), len(ops), t, buf, 148 * 16, C.byref(grid)))
    a = np.array(buf[:grid.value * 16], dtype=np.int64).reshape(grid.value, 16)[:, :16]
    # slot 0: globaltimer ns at CTA entry; slots 1-15: SM cycles since entry + 1 (ios.h)
    ghz = float(os.environ.get("IOS_SM_GHZ", "1.965"))
    if not (a[:, 0] > 0).any():
        print(f"stage {ops} T={t}: no trace stamps (grid {grid.value})")
        continue
    t0 = a[:, 0][a[:, 0] > 0].min()
    ent = (a[:, :1] - t0) / 1000.0
    rel = np.where(a > 0, ent + (a - 1) / (ghz * 1000.0), np.nan)
    rel[:, 0] = ent[:, 0]
    print(f"stage {ops} T={t} profiled {ms*1e3:.1f} us, grid {grid.value}; us since first entry (min/median/max over CTAs):")
    names = ["entry", "prologue", "P 1st issued", "P tile start", "mma done", "acc1 ready", "epi done", "teardown", "exit",
             "P expect_tx", "P A issued", "own prologue", "P 2nd issued", "e:13", "e:14", "e:15"]
    if os.environ.get("IOS_TRACE_FINE_NAMES"):   # libios built with -DIOS_TRACE_FINE
        names[13:16] = ["PDL wait done", "P tile decoded", "P TMA geom"]
    for k, nm in enumerate(names):
        col = rel[:, k]
        col = col[~np.isnan(col)]
        if len(col):
            print(f"   {nm:11s} {col.min():8.2f} {np.median(col):8.2f} {col.max():8.2f}  (n={len(col)})")
