"""O1/O2: the computation graph, groups, operator merge and schedule execution (TEST INFRASTRUCTURE ONLY).

* G = (V, E), edges are tensors. Ops run in insertion order, a topological order.
* Stage (S_i, T_i), T in {concurrent, merge}; Q = [(S_1,T_1)...(S_k,T_k)] runs in order.
* Groups: connected components of the stage's induced undirected subgraph (Z3).
* Merge: same-type convs with different hyper-parameters, kernels zero-padded to a common box and
  stacked, one conv, then a split (legality reading Z4).
"""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import tensor_ops as T

CONCURRENT, MERGE = 0, 1


class ScheduleError(ValueError):
    pass


class OracleGraph:
    def __init__(self, net):
        self.net = net
        self.ops = net.ops
        self.n = len(net.ops)
        self.shapes: Dict[int, Tuple[int, int, int, int]] = {0: tuple(net.input_shape)}
        for i in range(1, self.n + 1):
            self.shapes[i] = self._infer(i)
        # blocks: ordered list of block ids and their member ops (global ids, insertion order)
        self.block_ids: List[int] = []
        self.block_members: Dict[int, List[int]] = {}
        for i, o in enumerate(self.ops, start=1):
            if o.block not in self.block_members:
                self.block_ids.append(o.block)
                self.block_members[o.block] = []
            self.block_members[o.block].append(i)
        self.local = {}
        for b, mem in self.block_members.items():
            for li, g in enumerate(mem):
                self.local[g] = (b, li)
        # within-block successor masks (bit i = local index i)
        self.succ: Dict[int, List[int]] = {b: [0] * len(m) for b, m in self.block_members.items()}
        self.pred: Dict[int, List[int]] = {b: [0] * len(m) for b, m in self.block_members.items()}
        for v in range(1, self.n + 1):
            bv, lv = self.local[v]
            for u in self.ops[v - 1].inputs:
                if u == 0:
                    continue
                bu, lu = self.local[u]
                if bu == bv:
                    self.succ[bv][lu] |= 1 << lv
                    self.pred[bv][lv] |= 1 << lu
                elif self.block_ids.index(bu) > self.block_ids.index(bv):
                    raise ValueError("edge from a later block to an earlier block")

    # ---------------------------------------------------------------------------- shapes (O1)
    def _infer(self, i: int) -> Tuple[int, int, int, int]:
        o = self.ops[i - 1]
        n, c, h, w = self.shapes[o.inputs[0]]
        k = o.kind
        if k == "conv":
            return (n, o.cout, T.out_size(h, o.kh, o.sh, o.ph), T.out_size(w, o.kw, o.sw, o.pw))
        if k == "sepconv":
            return (n, o.cout, T.out_size(h, o.kh, o.sh, o.ph), T.out_size(w, o.kw, o.sw, o.pw))
        if k in ("maxpool", "avgpool"):
            return (n, c, T.out_size(h, o.kh, o.sh, o.ph, o.ceil_mode), T.out_size(w, o.kw, o.sw, o.pw, o.ceil_mode))
        if k == "gavgpool":
            return (n, c, 1, 1)
        if k in ("add", "identity"):
            for u in o.inputs:
                if self.shapes[u] != (n, c, h, w):
                    raise ValueError(f"op {i}: add/identity input shapes differ")
            return (n, c, h, w)
        if k == "concat":
            for u in o.inputs:
                if self.shapes[u][2:] != (h, w):
                    raise ValueError(f"op {i}: concat spatial shapes differ")
            return (n, sum(self.shapes[u][1] for u in o.inputs), h, w)
        if k == "linear":
            return (n, o.cout, 1, 1)
        raise ValueError(k)

    # ---------------------------------------------------------------------------- op execution
    def run_op(self, i: int, vals: Dict[int, np.ndarray]) -> np.ndarray:
        o = self.ops[i - 1]
        xs = [vals[u] for u in o.inputs]
        k = o.kind
        if k == "conv":
            x = T.relu(xs[0]) if o.relu_pre else xs[0]
            y = T.conv2d(x, o.weight, o.bias, o.sh, o.sw, o.ph, o.pw)
            return T.relu(y) if o.relu_post else y
        if k == "sepconv":
            return T.sepconv(xs, o.weight, o.bias, o.cout, o.kh, o.sh, o.ph, o.add_weights, o.relu_post)
        if k == "maxpool":
            return T.maxpool2d(xs[0], o.kh, o.sh, o.ph, o.ceil_mode)
        if k == "avgpool":
            return T.avgpool2d(xs[0], o.kh, o.sh, o.ph, o.count_include_pad, o.ceil_mode)
        if k == "gavgpool":
            return T.global_avgpool(xs[0], o.relu_pre)
        if k == "add":
            return T.add(xs, o.add_weights)
        if k == "concat":
            return T.concat(xs)
        if k == "identity":
            return np.array(xs[0], dtype=np.float64)
        if k == "linear":
            return T.linear(xs[0], o.weight, o.bias, o.relu_post)
        raise ValueError(k)

    def run_sequential(self, x: np.ndarray, keep: bool = True) -> Dict[int, np.ndarray]:
        """The sequential schedule: ops one by one in insertion (topological) order."""
        vals: Dict[int, np.ndarray] = {0: np.asarray(x, dtype=np.float64)}
        for i in range(1, self.n + 1):
            vals[i] = self.run_op(i, vals)
        return vals

    # ---------------------------------------------------------------------------- groups (Z3)
    def groups(self, block: int, mask: int) -> List[List[int]]:
        """Connected components of the induced undirected subgraph on ``mask``: local
        indices, each component in insertion order, components ordered by first member."""
        succ, pred = self.succ[block], self.pred[block]
        seen = 0
        comps = []
        for i in range(len(succ)):
            if not (mask >> i) & 1 or (seen >> i) & 1:
                continue
            comp = 1 << i
            frontier = [i]
            while frontier:
                u = frontier.pop()
                nb = (succ[u] | pred[u]) & mask & ~comp
                j = 0
                while nb:
                    if nb & 1:
                        comp |= 1 << j
                        frontier.append(j)
                    nb >>= 1
                    j += 1
            seen |= comp
            comps.append([j for j in range(len(succ)) if (comp >> j) & 1])
        return comps

    # ---------------------------------------------------------------------------- merge (Z4)
    def mergeable(self, ops: Sequence[int]) -> bool:
        """same type, hyper-parameters may differ; reading Z4: plain convs reading the
        identical input tensor, same stride and pre-ReLU, equal output H x W, |S'| >= 2."""
        if len(ops) < 2:
            return False
        os_ = [self.ops[i - 1] for i in ops]
        if any(o.kind != "conv" for o in os_):
            return False
        first = os_[0]
        for i, o in zip(ops, os_):
            if o.inputs[0] != first.inputs[0] or (o.sh, o.sw) != (first.sh, first.sw):
                return False
            if o.relu_pre != first.relu_pre or self.shapes[i][2:] != self.shapes[ops[0]][2:]:
                return False
        return True

    def merged_conv(self, ops: Sequence[int]):
        """Build the merged operator explicitly: bounding box of the members' windows on
        the common output grid, start = min(-p_i), end = max(-p_i + k_i); member i sits at offset
        (-p_i - start) with zeros elsewhere; filters stacked in the given order."""
        os_ = [self.ops[i - 1] for i in ops]
        st_h = min(-o.ph for o in os_)
        en_h = max(-o.ph + o.kh for o in os_)
        st_w = min(-o.pw for o in os_)
        en_w = max(-o.pw + o.kw for o in os_)
        kh, kw = en_h - st_h, en_w - st_w
        cin = os_[0].weight.shape[1]
        cout = sum(o.cout for o in os_)
        wm = np.zeros((cout, cin, kh, kw), dtype=np.float64)
        bm = np.zeros(cout, dtype=np.float64)
        c0 = 0
        splits = []
        for o in os_:
            oh, ow = -o.ph - st_h, -o.pw - st_w
            wm[c0:c0 + o.cout, :, oh:oh + o.kh, ow:ow + o.kw] = o.weight
            if o.bias is not None:
                bm[c0:c0 + o.cout] = o.bias
            splits.append((c0, c0 + o.cout))
            c0 += o.cout
        return wm, bm, (kh, kw), (-st_h, -st_w), splits

    def run_merged(self, ops: Sequence[int], vals: Dict[int, np.ndarray]) -> Dict[int, np.ndarray]:
        """ONE convolution with the merged kernel, then the split."""
        os_ = [self.ops[i - 1] for i in ops]
        wm, bm, (kh, kw), (ph, pw), splits = self.merged_conv(ops)
        x = vals[os_[0].inputs[0]]
        x = T.relu(x) if os_[0].relu_pre else x
        _, _, ho, wo = self.shapes[ops[0]]
        y = T.conv2d(x, wm, bm, os_[0].sh, os_[0].sw, ph, pw, ho=ho, wo=wo)
        out = {}
        for i, o, (a, b) in zip(ops, os_, splits):
            yi = y[:, a:b]
            out[i] = T.relu(yi) if o.relu_post else yi
        return out

    # ---------------------------------------------------------------------------- schedules (O2)
    def validate_schedule(self, q: Sequence[Tuple[Sequence[int], int]]) -> None:
        """Q is valid iff every op appears once and for every edge (u, v) either stage(u) <
        stage(v), or u, v share a concurrent stage's group with u earlier (each stage is then an
        ending of the ops not yet scheduled). Merge stages must be legal (Z4/Z5)."""
        stage_of: Dict[int, int] = {}
        for si, (ops, t) in enumerate(q):
            for v in ops:
                if v in stage_of or not (1 <= v <= self.n):
                    raise ScheduleError(f"op {v} repeated or unknown")
                stage_of[v] = si
            blocks = {self.local[v][0] for v in ops}
            if len(blocks) != 1:
                raise ScheduleError("stage spans blocks")
            if t == MERGE and not self.mergeable(list(ops)):
                raise ScheduleError("merge stage is not mergeable")
        if len(stage_of) != self.n:
            raise ScheduleError("schedule does not cover every op")
        for v in range(1, self.n + 1):
            for u in self.ops[v - 1].inputs:
                if u == 0:
                    continue
                su, sv = stage_of[u], stage_of[v]
                if su > sv or (su == sv and (q[su][1] == MERGE or u > v)):
                    raise ScheduleError(f"edge {u}->{v} violates the stage order")
        # blocks must run in order (per-block schedules are concatenated)
        order = [self.block_ids.index(self.local[q[si][0][0]][0]) for si in range(len(q))]
        if order != sorted(order):
            raise ScheduleError("blocks out of order")

    def run_schedule(self, q, x: np.ndarray, rng: Optional[np.random.Generator] = None) -> Dict[int, np.ndarray]:
        """Execute Q stage by stage. Concurrent stages run their groups in a random order
        (independence), group members in insertion order; merge stages run the explicit
        merged convolution."""
        self.validate_schedule(q)
        rng = rng if rng is not None else np.random.default_rng(0)
        vals: Dict[int, np.ndarray] = {0: np.asarray(x, dtype=np.float64)}
        for ops, t in q:
            ops = sorted(ops)
            if t == MERGE:
                vals.update(self.run_merged(ops, vals))
                continue
            b = self.local[ops[0]][0]
            mask = 0
            for v in ops:
                mask |= 1 << self.local[v][1]
            comps = self.groups(b, mask)
            for gi in rng.permutation(len(comps)):
                for li in comps[gi]:
                    v = self.block_members[b][li]
                    vals[v] = self.run_op(v, vals)
        return vals

    # ---------------------------------------------------------------------------- helpers
    def block_mask_ops(self, block: int, mask: int) -> List[int]:
        return [g for li, g in enumerate(self.block_members[block]) if (mask >> li) & 1]

    def flops(self, i: int) -> int:
        """2 * MACs of op i (conv / sepconv / linear; 0 otherwise), unpadded."""
        o = self.ops[i - 1]
        n, co, ho, wo = self.shapes[i]
        if o.kind == "conv":
            cin = self.shapes[o.inputs[0]][1]
            return 2 * n * ho * wo * co * cin * o.kh * o.kw
        if o.kind == "sepconv":
            c = self.shapes[o.inputs[0]][1]
            return 2 * n * ho * wo * c * (o.kh * o.kw + co)
        if o.kind == "linear":
            cin = int(np.prod(self.shapes[o.inputs[0]][1:]))
            return 2 * n * co * cin
        return 0
