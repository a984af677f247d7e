import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads as W
from paper_2011_01302_b200 import Graph
from paper_2011_01302_b200.ios import lib, _check, _i32
net = W.build("inception_v3"); g = Graph.from_netspec(net)
lib.ios_stage_trace.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.c_int32, C.c_int32, C.POINTER(C.c_uint64), C.c_int32, C.POINTER(C.c_int32)]
for rep in range(3):
    buf = (C.c_uint64 * (148 * 16))(); grid = C.c_int32()
    _check(lib.ios_stage_trace(g.handle, _i32([97]), 1, 0, buf, 148 * 16, C.byref(grid)))
    a = np.array(buf[:grid.value * 16], dtype=np.int64).reshape(grid.value, 16)
    print("load1 ns med", np.median(a[:, 13]), "load2 ns med", np.median(a[:, 14]), "10k cycles ns", np.median(a[:, 15]), "-> MHz", 1e4 / np.median(a[:, 15]) * 1e3)
