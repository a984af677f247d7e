"""Thin ctypes binding of libios (include/ios.h). Argument marshalling only: every step of the
stage executor runs in the library's CUDA kernels; there is no Python or CPU fallback and the
import fails loudly when libios.so is missing.

The module-level ``ios_*`` functions mirror the C-ABI one to one; ``Graph`` / ``Schedule`` are
conveniences built on them. PyTorch is used only for device memory and streams.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IOS_LIB") or os.path.join(_HERE, "libios.so")   # IOS_LIB: experiment builds

IOS_OK = 0
STATUS = {0: "IOS_OK", 1: "IOS_ERR_INVALID_ARG", 2: "IOS_ERR_DANGLING_INPUT", 3: "IOS_ERR_SHAPE", 4: "IOS_ERR_BLOCK",
          5: "IOS_ERR_NOT_MERGEABLE", 6: "IOS_ERR_NOT_A_STAGE", 7: "IOS_ERR_BAD_SCHEDULE", 8: "IOS_ERR_CUDA",
          9: "IOS_ERR_OOM", 10: "IOS_ERR_KERNEL", 11: "IOS_ERR_UNSUPPORTED"}
MATH = {"tf32": 0, "bf16": 1, "fp32_simt": 2}
CONCURRENT, MERGE = 0, 1
STRATEGY_SETS = {"both": 0, "merge": 1, "parallel": 2}
OP_KIND = {"conv": 0, "sepconv": 1, "maxpool": 2, "avgpool": 3, "gavgpool": 4, "add": 5, "concat": 6,
           "identity": 7, "linear": 8}
F_RELU_POST, F_RELU_PRE, F_CEIL_MODE, F_COUNT_INCLUDE_PAD = 1, 2, 4, 8


class IOSError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class OpDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("block", C.c_int32), ("out_channels", C.c_int32),
                ("kernel_h", C.c_int32), ("kernel_w", C.c_int32), ("stride_h", C.c_int32), ("stride_w", C.c_int32),
                ("pad_h", C.c_int32), ("pad_w", C.c_int32), ("flags", C.c_int32),
                ("weight", C.POINTER(C.c_float)), ("bias", C.POINTER(C.c_float)),
                ("add_weights", C.POINTER(C.c_float))]


class ProfileOpts(C.Structure):
    _fields_ = [("warmup", C.c_int32), ("trials", C.c_int32), ("reps", C.c_int32), ("l2_flush", C.c_int32)]


COST_FN = C.CFUNCTYPE(C.c_double, C.c_void_p, C.c_int32, C.c_uint64, C.c_int)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(the stage executor has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P, I32, I64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    pI32, pD = C.POINTER(I32), C.POINTER(D)
    sig = {
        "ios_graph_create": [I32, I32, I32, I32, I32, I32, C.POINTER(P)],
        "ios_add_op": [P, C.POINTER(OpDesc), pI32, I32, pI32],
        "ios_graph_num_ops": [P, pI32],
        "ios_op_shape": [P, I32, pI32],
        "ios_graph_num_blocks": [P, pI32],
        "ios_graph_block_ops": [P, I32, pI32, I32, pI32, pI32],
        "ios_stage_mergeable": [P, pI32, I32, pI32],
        "ios_stage_latency": [P, pI32, I32, I32, C.POINTER(ProfileOpts), pD],
        "ios_schedule_dp": [P, I32, I32, COST_FN, P, C.POINTER(P), pD],
        "ios_schedule_dp_ex": [P, I32, I32, I32, COST_FN, P, C.POINTER(P), pD, C.POINTER(I64)],
        "ios_schedule_sequential": [P, C.POINTER(P)],
        "ios_schedule_greedy": [P, C.POINTER(P)],
        "ios_schedule_create": [P, I32, pI32, pI32, pI32, C.POINTER(P)],
        "ios_schedule_num_stages": [P, pI32],
        "ios_schedule_stage": [P, I32, pI32, I32, pI32, pI32, pD],
        "ios_schedule_tune": [P, P, I32, I32],
        "ios_run": [P, P, P, P, P],
        "ios_run_host": [P, P, C.POINTER(C.c_float), C.POINTER(C.c_float), P],
        "ios_op_output": [P, I32, P, P],
        "ios_schedule_launches": [P, P, pI32],
        "ios_latency_cache_save": [P, C.c_char_p],
        "ios_latency_cache_load": [P, C.c_char_p],
        "ios_latency_cache_autosave": [P, C.c_char_p],
        "ios_sync": [P, P],
        "ios_schedule_refine": [P, I32, I32, I32, D, C.POINTER(P), C.POINTER(I64)],
        "ios_tile_variants_save": [P, C.c_char_p],
        "ios_tile_variants_load": [P, C.c_char_p],
        "ios_run_timeline": [P, P, P, P, I32, I32, pD, I32],
    }
    for name, args in sig.items():
        if os.environ.get("IOS_LIB") and not hasattr(lib, name):
            continue   # an older experiment build (A/B runs) may lack newer entry points
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = I32
    lib.ios_last_error.restype = C.c_char_p
    lib.ios_last_error.argtypes = []
    if hasattr(lib, "ios_build_id"):
        lib.ios_build_id.restype = C.c_char_p
        lib.ios_build_id.argtypes = []
    lib.ios_schedule_destroy.argtypes = [P]
    lib.ios_schedule_destroy.restype = None
    lib.ios_graph_destroy.argtypes = [P]
    lib.ios_graph_destroy.restype = None
    return lib


lib = _load()


def _check(st: int) -> None:
    if st != IOS_OK:
        raise IOSError(st, (lib.ios_last_error() or b"").decode())


def _i32(seq: Sequence[int]):
    return (C.c_int32 * max(1, len(seq)))(*[int(v) for v in seq])


def _fptr(a: Optional[np.ndarray]):
    if a is None:
        return None, None
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a, a.ctypes.data_as(C.POINTER(C.c_float))


# ---------------------------------------------------------------------------- 1:1 ABI functions
def ios_graph_create(batch: int, c: int, h: int, w: int, math_mode: str = "tf32", device: int = 0) -> C.c_void_p:
    g = C.c_void_p()
    _check(lib.ios_graph_create(batch, c, h, w, MATH[math_mode], device, C.byref(g)))
    return g


def ios_add_op(g, kind: str, inputs: Sequence[int], block: int, out_channels: int = 0, kernel=(1, 1), stride=(1, 1),
               pad=(0, 0), flags: int = 0, weight=None, bias=None, add_weights=None) -> int:
    wk, wp = _fptr(weight)
    bk, bp = _fptr(bias)
    ak, ap = _fptr(add_weights)
    d = OpDesc(OP_KIND[kind], block, out_channels, kernel[0], kernel[1], stride[0], stride[1], pad[0], pad[1], flags,
               wp, bp, ap)
    out = C.c_int32()
    _check(lib.ios_add_op(g, C.byref(d), _i32(inputs), len(inputs), C.byref(out)))
    return out.value


def ios_stage_latency(g, ops: Sequence[int], strategy: int = CONCURRENT, warmup: int = 0, trials: int = 0,
                      reps: int = 0, l2_flush: bool = False) -> float:
    o = ProfileOpts(warmup, trials, reps, int(l2_flush))
    ms = C.c_double()
    _check(lib.ios_stage_latency(g, _i32(ops), len(ops), strategy, C.byref(o), C.byref(ms)))
    return ms.value


def ios_schedule_dp(g, r: int, s: int, cost: Optional[Callable[[int, int, int], float]] = None,
                    strategies: str = "both"):
    """Returns (schedule handle, cost ms, (states, transitions, distinct stages costed))."""
    if cost is None:
        cb = C.cast(None, COST_FN)
    else:
        cb = COST_FN(lambda ctx, block, mask, t: float(cost(int(block), int(mask), int(t))))
    q = C.c_void_p()
    tot = C.c_double()
    stats = (C.c_int64 * 3)()
    _check(lib.ios_schedule_dp_ex(g, r, s, STRATEGY_SETS[strategies], cb, None, C.byref(q), C.byref(tot), stats))
    return q, tot.value, tuple(int(v) for v in stats)


def ios_schedule_tune(g, q, trials: int = 0, reps: int = 0) -> None:
    _check(lib.ios_schedule_tune(g, q, trials, reps))


def ios_run(g, q, d_input: int, d_output: int, stream: int = 0) -> None:
    _check(lib.ios_run(g, q, C.c_void_p(d_input), C.c_void_p(d_output), C.c_void_p(stream)))


def ios_last_error() -> str:
    return (lib.ios_last_error() or b"").decode()


def ios_sync(g, stream: int = 0) -> None:
    """Synchronise `stream`; IOS_ERR_KERNEL if an in-kernel dependency wait of an earlier run timed out."""
    _check(lib.ios_sync(g, C.c_void_p(stream)))


def ios_build_id() -> str:
    return (lib.ios_build_id() or b"").decode()


# ---------------------------------------------------------------------------- conveniences
class Schedule:
    def __init__(self, graph: "Graph", handle: C.c_void_p, cost: Optional[float] = None, stats=None):
        self.graph = graph
        self.handle = handle
        self.cost = cost
        self.stats = stats

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and lib is not None:
            lib.ios_schedule_destroy(h)
            self.handle = None

    @property
    def stages(self) -> List[Tuple[List[int], int, float]]:
        n = C.c_int32()
        _check(lib.ios_schedule_num_stages(self.handle, C.byref(n)))
        out = []
        for i in range(n.value):
            cap = 64
            ops = (C.c_int32 * cap)()
            k = C.c_int32()
            t = C.c_int32()
            lat = C.c_double()
            _check(lib.ios_schedule_stage(self.handle, i, ops, cap, C.byref(k), C.byref(t), C.byref(lat)))
            out.append(([ops[j] for j in range(k.value)], t.value, lat.value))
        return out

    def launches(self) -> int:
        n = C.c_int32()
        _check(lib.ios_schedule_launches(self.graph.handle, self.handle, C.byref(n)))
        return n.value


class Graph:
    """An ``ios_graph`` plus the NetSpec-like bookkeeping needed to marshal inputs/outputs."""

    def __init__(self, batch: int, c: int, h: int, w: int, math_mode: str = "tf32", device: int = 0):
        self.handle = ios_graph_create(batch, c, h, w, math_mode, device)
        self.math = math_mode
        self.device = device
        self.input_shape = (batch, c, h, w)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and lib is not None:
            lib.ios_graph_destroy(h)
            self.handle = None

    @classmethod
    def from_netspec(cls, net, math_mode: Optional[str] = None, device: int = 0) -> "Graph":
        g = cls(*net.input_shape, math_mode or net.math, device)
        for i, o in enumerate(net.ops, start=1):
            oid = ios_add_op(g.handle, o.kind, o.inputs, o.block, o.cout, (o.kh, o.kw), (o.sh, o.sw), (o.ph, o.pw),
                             o.flags(), o.weight, o.bias, o.add_weights)
            assert oid == i
        return g

    # -- structure
    @property
    def num_ops(self) -> int:
        n = C.c_int32()
        _check(lib.ios_graph_num_ops(self.handle, C.byref(n)))
        return n.value

    def op_shape(self, op: int) -> Tuple[int, int, int, int]:
        s = (C.c_int32 * 4)()
        _check(lib.ios_op_shape(self.handle, op, s))
        return tuple(s)

    def blocks(self) -> List[Tuple[int, List[int]]]:
        nb = C.c_int32()
        _check(lib.ios_graph_num_blocks(self.handle, C.byref(nb)))
        out = []
        for b in range(nb.value):
            ops = (C.c_int32 * 64)()
            n = C.c_int32()
            bid = C.c_int32()
            _check(lib.ios_graph_block_ops(self.handle, b, ops, 64, C.byref(n), C.byref(bid)))
            out.append((bid.value, [ops[i] for i in range(n.value)]))
        return out

    def mergeable(self, ops: Sequence[int]) -> bool:
        m = C.c_int32()
        _check(lib.ios_stage_mergeable(self.handle, _i32(ops), len(ops), C.byref(m)))
        return bool(m.value)

    # -- measurement / scheduling
    def stage_latency(self, ops: Sequence[int], strategy: int = CONCURRENT, **kw) -> float:
        return ios_stage_latency(self.handle, ops, strategy, **kw)

    def schedule_dp(self, r: int = 3, s: int = 8, cost=None, strategies: str = "both") -> Schedule:
        q, c, stats = ios_schedule_dp(self.handle, r, s, cost, strategies)
        return Schedule(self, q, c, stats)

    def schedule_refine(self, r: int = 3, s: int = 8, reps: int = 10, beta_us: float = 1.0) -> Schedule:
        """ios_schedule_refine: DP optima under a family of cost models, chosen per block in context."""
        q = C.c_void_p()
        stats = (C.c_int64 * 4)()
        _check(lib.ios_schedule_refine(self.handle, r, s, reps, beta_us, C.byref(q), stats))
        return Schedule(self, q, None, tuple(int(v) for v in stats))

    def tune(self, q: Schedule, trials: int = 0, reps: int = 0) -> None:
        """ios_schedule_tune: pick each stage's tiling variant by measurement (call before runs)."""
        ios_schedule_tune(self.handle, q.handle, trials, reps)

    def schedule_sequential(self) -> Schedule:
        q = C.c_void_p()
        _check(lib.ios_schedule_sequential(self.handle, C.byref(q)))
        return Schedule(self, q)

    def schedule_greedy(self) -> Schedule:
        q = C.c_void_p()
        _check(lib.ios_schedule_greedy(self.handle, C.byref(q)))
        return Schedule(self, q)

    def schedule(self, stages: Sequence[Tuple[Sequence[int], int]]) -> Schedule:
        sizes = [len(s[0]) for s in stages]
        ops = [v for s in stages for v in s[0]]
        strat = [int(s[1]) for s in stages]
        q = C.c_void_p()
        _check(lib.ios_schedule_create(self.handle, len(stages), _i32(sizes), _i32(ops), _i32(strat), C.byref(q)))
        return Schedule(self, q)

    # -- execution (torch is used only for device memory and streams)
    def output_shape(self) -> Tuple[int, int, int, int]:
        return self.op_shape(self.num_ops)

    def run(self, q: Schedule, x, out=None, stream=None):
        import torch
        assert x.is_cuda and x.dtype == torch.float32 and x.is_contiguous()
        if out is None:
            out = torch.empty(self.output_shape(), dtype=torch.float32, device=x.device)
        st = stream if stream is not None else torch.cuda.current_stream(x.device).cuda_stream
        ios_run(self.handle, q.handle, x.data_ptr(), out.data_ptr(), st)
        return out

    def run_host(self, q: Schedule, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float32)
        out = np.empty(self.output_shape(), dtype=np.float32)
        _check(lib.ios_run_host(self.handle, q.handle, x.ctypes.data_as(C.POINTER(C.c_float)),
                                out.ctypes.data_as(C.POINTER(C.c_float)), None))
        return out

    def run_timeline(self, q: Schedule, x, out=None, reps: int = 10, l2_flush: bool = True):
        """ios_run_timeline: per stage (start_us, end_us, attributable_us), mean over `reps` runs."""
        import torch
        if out is None:
            out = torch.empty(self.output_shape(), dtype=torch.float32, device=x.device)
        n = len(q.stages)
        buf = (C.c_double * (3 * max(1, n)))()
        _check(lib.ios_run_timeline(self.handle, q.handle, C.c_void_p(x.data_ptr()), C.c_void_p(out.data_ptr()),
                                    reps, int(l2_flush), buf, 3 * max(1, n)))
        return [(buf[3 * i], buf[3 * i + 1], buf[3 * i + 2]) for i in range(n)]

    def sync(self, stream=None) -> None:
        """ios_sync on `stream` (default: torch's current stream of the graph's device)."""
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(torch.device(f"cuda:{self.device}")).cuda_stream
        ios_sync(self.handle, stream)

    def op_output(self, op: int, stream=None):
        import torch
        t = torch.empty(self.op_shape(op), dtype=torch.float32, device=f"cuda:{self.device}")
        st = stream if stream is not None else torch.cuda.current_stream(t.device).cuda_stream
        _check(lib.ios_op_output(self.handle, op, C.c_void_p(t.data_ptr()), C.c_void_p(st)))
        return t

    def save_tile_variants(self, path: str) -> None:
        _check(lib.ios_tile_variants_save(self.handle, path.encode()))

    def load_tile_variants(self, path: str) -> None:
        _check(lib.ios_tile_variants_load(self.handle, path.encode()))

    def save_latency_cache(self, path: str) -> None:
        _check(lib.ios_latency_cache_save(self.handle, path.encode()))

    def load_latency_cache(self, path: str) -> None:
        _check(lib.ios_latency_cache_load(self.handle, path.encode()))

    def autosave_latency_cache(self, path: str) -> None:
        """Checkpoint the stage-latency cache after every searched block (resume long searches)."""
        _check(lib.ios_latency_cache_autosave(self.handle, path.encode()))
