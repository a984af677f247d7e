"""O3: schedule search, written as Algorithm 1 — TEST INFRASTRUCTURE ONLY.

State S and ending S' are bit masks over one block's ops (bit i = i-th op of the block in
insertion order). ``cost_fn(block, mask, strategy) -> ms`` is the stage latency L(S', T): on the
device for the product, a fixed table in tests (Z8).

Readings: Z1 endings enumerated in canonical order (|S'| ascending, then mask
descending), first minimiser wins (strict < at L19); Z2 strategy tie -> merge (strict < at L30);
Z7 pruning P(r, s) counts connectivity groups of S' whatever the strategy.
"""
from __future__ import annotations

import math
from typing import Callable, Dict, List, Optional, Sequence, Tuple

CONCURRENT, MERGE = 0, 1
BOTH, MERGE_ONLY, PARALLEL_ONLY = 0, 1, 2   # IOS-Both / IOS-Merge / IOS-Parallel
INF = math.inf


def popcount(m: int) -> int:
    return bin(m).count("1")


def submasks(s: int):
    sub = s
    while sub:
        yield sub
        sub = (sub - 1) & s


def is_ending(succ: Sequence[int], s: int, sp: int) -> bool:
    """S' is an ending of S iff no edge goes from S' to S - S'."""
    rest = s & ~sp
    for i in range(len(succ)):
        if (sp >> i) & 1 and succ[i] & rest:
            return False
    return True


def components(succ: Sequence[int], pred: Sequence[int], sp: int) -> List[int]:
    """Connected components (as masks) of the undirected subgraph induced by S'."""
    comps = []
    left = sp
    while left:
        i = (left & -left).bit_length() - 1
        comp = 1 << i
        frontier = [i]
        while frontier:
            u = frontier.pop()
            nb = (succ[u] | pred[u]) & sp & ~comp
            while nb:
                j = (nb & -nb).bit_length() - 1
                nb &= nb - 1
                comp |= 1 << j
                frontier.append(j)
        comps.append(comp)
        left &= ~comp
    return comps


def satisfies_pruning(succ, pred, sp: int, r: Optional[int], s: Optional[int]) -> bool:
    """P(S, S') = True iff S' has at most s groups and each group has at most r ops."""
    if r is None and s is None:
        return True
    comps = components(succ, pred, sp)
    if s is not None and len(comps) > s:
        return False
    if r is not None and any(popcount(c) > r for c in comps):
        return False
    return True


def endings(succ, pred, s: int, r: Optional[int] = None, smax: Optional[int] = None) -> List[int]:
    """All non-empty endings of S satisfying P(r, s), in canonical order (Z1)."""
    out = [sp for sp in submasks(s) if is_ending(succ, s, sp) and satisfies_pruning(succ, pred, sp, r, smax)]
    out.sort(key=lambda m: (popcount(m), -m))
    return out


class BlockDP:
    """Algorithm 1 for one block (per-block optimisation)."""

    def __init__(self, succ: Sequence[int], pred: Sequence[int], cost_fn: Callable[[int, int], float],
                 mergeable: Callable[[int], bool], r: Optional[int] = None, s: Optional[int] = None,
                 strategies: int = BOTH):
        self.succ, self.pred = list(succ), list(pred)
        self.n = len(succ)
        self.cost_fn = cost_fn            # (mask, strategy) -> ms
        self.mergeable = mergeable        # mask -> bool
        self.r, self.s = r, s
        self.strategies = strategies
        self.cost: Dict[int, float] = {0: 0.0}                # L1: cost[empty] = 0, others = inf
        self.choice: Dict[int, Tuple[int, int]] = {}           # L2
        self.transitions = 0

    def generate_stage(self, sp: int) -> Tuple[float, int]:
        """L23-33: L_concurrent measured for the group partition; L_merge if mergeable else inf;
        concurrent iff L_concurrent < L_merge (ties -> merge)."""
        if self.strategies == MERGE_ONLY and popcount(sp) > 1:
            l_conc = INF
        else:
            l_conc = self.cost_fn(sp, CONCURRENT)                         # L24-25
        if self.strategies != PARALLEL_ONLY and self.mergeable(sp):       # L26
            l_merge = self.cost_fn(sp, MERGE)                             # L27
        else:
            l_merge = INF                                                 # L28-29
        if l_conc < l_merge:                                              # L30
            return l_conc, CONCURRENT                                     # L31
        return l_merge, MERGE                                             # L32-33

    def scheduler(self, s: int) -> float:
        """L13-22 (memoised recursion over states)."""
        if s in self.cost:                                                # L14-15
            return self.cost[s]
        best = INF
        for sp in endings(self.succ, self.pred, s, self.r, self.s):       # L16
            self.transitions += 1
            l_sp, t_sp = self.generate_stage(sp)                          # L17
            l_s = self.scheduler(s & ~sp) + l_sp                          # L18
            if l_s < best:                                                # L19
                best = l_s                                                # L20
                self.choice[s] = (sp, t_sp)                               # L21
        self.cost[s] = best
        return best                                                       # L22

    def run(self) -> Tuple[float, List[Tuple[int, int]]]:
        """L3-12: Scheduler(V) then rebuild Q by inserting choice[S] at the head."""
        v = (1 << self.n) - 1                                             # L4
        total = self.scheduler(v)                                         # L5
        q: List[Tuple[int, int]] = []                                     # L6
        s = v                                                             # L7
        while s:                                                          # L8
            sp, t = self.choice[s]                                        # L9
            q.insert(0, (sp, t))                                          # L10
            s &= ~sp                                                      # L11
        return total, q                                                   # L12


def dp(graph, cost_fn: Callable[[int, int, int], float], r: Optional[int] = 3, s: Optional[int] = 8,
       strategies: int = BOTH):
    """IOS over a whole OracleGraph: one DP per block, schedules concatenated in block order.
    Returns (total, Q) with Q = [(global op ids, strategy)], total = left fold of the block costs."""
    total = 0.0
    q: List[Tuple[List[int], int]] = []
    for b in graph.block_ids:
        mem = graph.block_members[b]
        bdp = BlockDP(graph.succ[b], graph.pred[b], lambda m, t, b=b: cost_fn(b, m, t),
                      lambda m, b=b: graph.mergeable(graph.block_mask_ops(b, m)), r, s, strategies)
        c, bq = bdp.run()
        total += c
        q.extend(([mem[i] for i in range(len(mem)) if (m >> i) & 1], t) for m, t in bq)
    return total, q


def all_schedules(succ, pred, mergeable: Callable[[int], bool], r=None, s=None):
    """Every schedule of a block: each peel sequence of endings x each legal strategy per stage,
    listed in execution order. Exponential: tiny graphs only (<= ~8 ops)."""
    n = len(succ)

    def rec(rem: int):
        if rem == 0:
            yield []
            return
        for sp in endings(succ, pred, rem, r, s):
            strategies = [CONCURRENT] + ([MERGE] if mergeable(sp) else [])
            for prefix in rec(rem & ~sp):
                for t in strategies:
                    yield prefix + [(sp, t)]

    yield from rec((1 << n) - 1)


def brute_force(succ, pred, cost_fn: Callable[[int, int], float], mergeable: Callable[[int], bool],
                r=None, s=None) -> Tuple[float, List[Tuple[int, int]]]:
    """Minimum over all schedules of the cost summed left to right in execution order."""
    best, best_q = INF, None
    for q in all_schedules(succ, pred, mergeable, r, s):
        c = 0.0
        for sp, t in q:
            c = c + cost_fn(sp, t)
        if c < best:
            best, best_q = c, q
    return best, best_q


def sequential(graph) -> List[Tuple[List[int], int]]:
    """One op per stage in insertion (topological) order (Z16)."""
    return [([i], CONCURRENT) for i in range(1, graph.n + 1)]


def greedy(graph) -> List[Tuple[List[int], int]]:
    """Repeatedly put every ready op of the block into one concurrent stage."""
    q = []
    for b in graph.block_ids:
        mem = graph.block_members[b]
        pred = graph.pred[b]
        rem = (1 << len(mem)) - 1
        while rem:
            ready = 0
            for i in range(len(mem)):
                if (rem >> i) & 1 and not (pred[i] & rem):
                    ready |= 1 << i
            q.append(([mem[i] for i in range(len(mem)) if (ready >> i) & 1], CONCURRENT))
            rem &= ~ready
    return q


def count(succ, pred, r=None, s=None) -> Tuple[int, int, int]:
    """(#states reachable from V incl. the empty set, #transitions (S, S') with S' a non-empty
    ending, #schedules = #paths V -> empty) — the quantities of Fig. 5 and Table 1."""
    n = len(succ)
    memo: Dict[int, int] = {0: 1}
    trans = [0]

    def paths(st: int) -> int:
        if st in memo:
            return memo[st]
        tot = 0
        for sp in endings(succ, pred, st, r, s):
            trans[0] += 1
            tot += paths(st & ~sp)
        memo[st] = tot
        return tot

    npaths = paths((1 << n) - 1)
    return len(memo), trans[0], npaths
