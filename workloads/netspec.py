"""Graph descriptions: G = (V, E) as an ordered op list ("Computation Graph").

Op ids: 0 is the graph input; op i (i >= 1) is ``ops[i-1]``. Every op's inputs are existing ids,
so insertion order is a topological order (the sequential schedule's order).
Each op carries a block id; the DP runs per block.

Weights follow DESIGN.md reading Z12: W ~ N(0, 2/fan_in) (He), b ~ U(-0.1, 0.1), one NumPy
``default_rng`` per op seeded from (net seed, op id). Nothing here computes on tensors.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple, Union

import numpy as np

OP_KINDS = ("conv", "sepconv", "maxpool", "avgpool", "gavgpool", "add", "concat", "identity", "linear")


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round fp32 values to the nearest bf16 (RNE) and return them as fp32 (Z14)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    out = (r & 0xFFFFFFFF).astype(np.uint32).view(np.float32)
    nan = np.isnan(a)
    if nan.any():
        out = out.copy()
        out[nan] = np.nan
    return out.reshape(a.shape)


@dataclass
class OpSpec:
    kind: str
    inputs: List[int]
    block: int
    cout: int = 0
    kh: int = 1
    kw: int = 1
    sh: int = 1
    sw: int = 1
    ph: int = 0
    pw: int = 0
    relu_post: bool = False
    relu_pre: bool = False
    ceil_mode: bool = False
    count_include_pad: bool = True
    weight: Optional[np.ndarray] = None       # conv [Cout][Cin][kh][kw]; sepconv dw [C][kh][kw] ++ pw [Cout][C]; linear [Cout][Cin]
    bias: Optional[np.ndarray] = None         # [Cout]
    add_weights: Optional[np.ndarray] = None  # add / sepconv aggregation weights [n_inputs]
    name: str = ""

    def flags(self) -> int:
        """Bit flags of the C-ABI (include/ios.h): RELU_POST=1, RELU_PRE=2, CEIL_MODE=4, COUNT_INCLUDE_PAD=8."""
        return (1 if self.relu_post else 0) | (2 if self.relu_pre else 0) | \
               (4 if self.ceil_mode else 0) | (8 if self.count_include_pad else 0)


@dataclass
class NetSpec:
    name: str
    input_shape: Tuple[int, int, int, int]   # N, C, H, W
    ops: List[OpSpec] = field(default_factory=list)
    seed: int = 0
    math: str = "tf32"                        # the configuration's compute mode (BASELINE.json configs)

    @property
    def n_ops(self) -> int:
        return len(self.ops)

    @property
    def output_id(self) -> int:
        return len(self.ops)

    def op(self, i: int) -> OpSpec:
        return self.ops[i - 1]

    def blocks(self) -> List[int]:
        seen: List[int] = []
        for o in self.ops:
            if not seen or seen[-1] != o.block:
                seen.append(o.block)
        return seen

    def block_ops(self, b: int) -> List[int]:
        return [i + 1 for i, o in enumerate(self.ops) if o.block == b]

    def make_input(self, seed: int = 1234, batch: Optional[int] = None) -> np.ndarray:
        """x ~ N(0, 1) fp32 NCHW (SURVEY §8d "Concrete synthetic inputs")."""
        n, c, h, w = self.input_shape
        if batch is not None:
            n = batch
        rng = np.random.default_rng(seed)
        x = rng.standard_normal((n, c, h, w)).astype(np.float32)
        return bf16_round(x) if self.math == "bf16" else x

    def with_batch(self, batch: int) -> "NetSpec":
        n, c, h, w = self.input_shape
        return NetSpec(self.name, (batch, c, h, w), self.ops, self.seed, self.math)


Int2 = Union[int, Tuple[int, int]]


def _pair(v: Int2) -> Tuple[int, int]:
    return (v, v) if isinstance(v, int) else (int(v[0]), int(v[1]))


class NetBuilder:
    """Appends ops in topological order; tracks channel counts only (to size weights)."""

    def __init__(self, name: str, input_shape: Sequence[int], seed: int = 0, math: str = "tf32"):
        self.net = NetSpec(name, tuple(int(v) for v in input_shape), [], seed, math)
        self.ch = {0: int(input_shape[1])}
        self.block = 0

    # -- helpers -----------------------------------------------------------------------------
    def new_block(self) -> int:
        if self.net.ops and self.net.ops[-1].block == self.block:
            self.block += 1
        return self.block

    def _rng(self) -> np.random.Generator:
        return np.random.default_rng([self.net.seed, len(self.net.ops) + 1])

    def _push(self, op: OpSpec, cout: int) -> int:
        if self.net.math == "bf16":
            for attr in ("weight", "bias", "add_weights"):
                v = getattr(op, attr)
                if v is not None:
                    setattr(op, attr, bf16_round(v))
        self.net.ops.append(op)
        i = len(self.net.ops)
        self.ch[i] = cout
        return i

    # -- ops -----------------------------------------------------------------------------------
    def conv(self, x: int, cout: int, k: Int2, s: Int2 = 1, p: Int2 = 0, relu: bool = True,
             relu_pre: bool = False, bias: bool = True, name: str = "") -> int:
        kh, kw = _pair(k)
        sh, sw = _pair(s)
        ph, pw = _pair(p)
        cin = self.ch[x]
        rng = self._rng()
        w = (rng.standard_normal((cout, cin, kh, kw)) * np.sqrt(2.0 / (cin * kh * kw))).astype(np.float32)
        b = rng.uniform(-0.1, 0.1, cout).astype(np.float32) if bias else None
        return self._push(OpSpec("conv", [x], self.block, cout, kh, kw, sh, sw, ph, pw,
                                 relu_post=relu, relu_pre=relu_pre, weight=w, bias=b, name=name), cout)

    def sepconv(self, xs: Union[int, Sequence[int]], cout: int, k: int, s: int = 1, p: Optional[int] = None,
                add_weights: Optional[Sequence[float]] = None, relu_post: bool = False, name: str = "") -> int:
        """Relu-SepConv unit (Table 2): [weighted sum of inputs] -> ReLU -> dw k x k -> pw 1x1 (+bias)."""
        xs = [xs] if isinstance(xs, int) else list(xs)
        cin = self.ch[xs[0]]
        assert all(self.ch[v] == cin for v in xs)
        p = k // 2 if p is None else p
        rng = self._rng()
        dw = (rng.standard_normal((cin, k, k)) * np.sqrt(2.0 / (k * k))).astype(np.float32)
        pw = (rng.standard_normal((cout, cin)) * np.sqrt(2.0 / cin)).astype(np.float32)
        b = rng.uniform(-0.1, 0.1, cout).astype(np.float32)
        wts = None
        if len(xs) > 1:
            wts = np.asarray(add_weights if add_weights is not None else np.ones(len(xs)), dtype=np.float32)
        w = np.concatenate([dw.ravel(), pw.ravel()]).astype(np.float32)
        return self._push(OpSpec("sepconv", xs, self.block, cout, k, k, s, s, p, p, relu_post=relu_post,
                                 relu_pre=True, weight=w, bias=b, add_weights=wts, name=name), cout)

    def maxpool(self, x: int, k: int, s: int, p: int = 0, ceil_mode: bool = False, name: str = "") -> int:
        c = self.ch[x]
        return self._push(OpSpec("maxpool", [x], self.block, c, k, k, s, s, p, p, ceil_mode=ceil_mode,
                                 count_include_pad=False, name=name), c)

    def avgpool(self, x: int, k: int, s: int, p: int = 0, count_include_pad: bool = True,
                ceil_mode: bool = False, name: str = "") -> int:
        c = self.ch[x]
        return self._push(OpSpec("avgpool", [x], self.block, c, k, k, s, s, p, p, ceil_mode=ceil_mode,
                                 count_include_pad=count_include_pad, name=name), c)

    def gavgpool(self, x: int, relu_pre: bool = False, name: str = "") -> int:
        c = self.ch[x]
        return self._push(OpSpec("gavgpool", [x], self.block, c, relu_pre=relu_pre, name=name), c)

    def add(self, xs: Sequence[int], weights: Optional[Sequence[float]] = None, name: str = "") -> int:
        c = self.ch[xs[0]]
        assert all(self.ch[v] == c for v in xs)
        wts = None if weights is None else np.asarray(weights, dtype=np.float32)
        return self._push(OpSpec("add", list(xs), self.block, c, add_weights=wts, name=name), c)

    def concat(self, xs: Sequence[int], name: str = "") -> int:
        c = sum(self.ch[v] for v in xs)
        return self._push(OpSpec("concat", list(xs), self.block, c, name=name), c)

    def identity(self, x: int, name: str = "") -> int:
        c = self.ch[x]
        return self._push(OpSpec("identity", [x], self.block, c, name=name), c)

    def linear(self, x: int, cout: int, relu: bool = False, name: str = "") -> int:
        cin = self.ch[x]
        rng = self._rng()
        w = (rng.standard_normal((cout, cin)) * np.sqrt(1.0 / cin)).astype(np.float32)
        b = rng.uniform(-0.1, 0.1, cout).astype(np.float32)
        return self._push(OpSpec("linear", [x], self.block, cout, relu_post=relu, weight=w, bias=b, name=name), cout)
