"""Seeded random DAGs and fixed stage-cost tables for schedule-search tests.

A cost table stands in for the device ("fake device"): a deterministic function
(block, stage mask, strategy) -> milliseconds. The same Python callable is handed to the oracle
DP and (through the C-ABI ``ios_cost_fn`` callback) to the library's DP, so any schedule
difference is a search difference, never a cost difference.
"""
from __future__ import annotations

import hashlib
import struct
from typing import Callable, List, Sequence

import numpy as np

from .netspec import NetBuilder, NetSpec

CONCURRENT, MERGE = 0, 1


def random_dag(n: int, p: float, seed: int) -> List[List[int]]:
    """Predecessor lists of a random DAG on nodes 0..n-1 (edges only from lower to higher index)."""
    rng = np.random.default_rng([seed, n, int(p * 1000)])
    return [sorted(int(u) for u in range(v) if rng.random() < p) for v in range(n)]


def dag_net(preds: Sequence[Sequence[int]], channels: int = 8, hw: int = 4, seed: int = 0,
            conv_k: int = 1) -> NetSpec:
    """A NetSpec whose block 0 has exactly the DAG's edges: a node with 0 predecessors is a conv on
    the graph input, with 1 predecessor a conv on it, with >= 2 an add of them."""
    nb = NetBuilder("dag", (1, channels, hw, hw), seed)
    ids: List[int] = []
    for v, ps in enumerate(preds):
        if len(ps) == 0:
            ids.append(nb.conv(0, channels, conv_k, 1, conv_k // 2, name=f"n{v}"))
        elif len(ps) == 1:
            ids.append(nb.conv(ids[ps[0]], channels, conv_k, 1, conv_k // 2, name=f"n{v}"))
        else:
            ids.append(nb.add([ids[u] for u in ps], name=f"n{v}"))
    return nb.net


def _u01(*key) -> float:
    h = hashlib.blake2b(struct.pack(f"<{len(key)}q", *key), digest_size=8).digest()
    return int.from_bytes(h, "little") / 2.0 ** 64


def random_cost_table(seed: int, merge_frac: float = 1.0) -> Callable[[int, int, int], float]:
    """cost(block, mask, strategy) -> float ms: a fixed pseudo-random (non-dyadic) table. Merge
    costs are finite for the strategies the caller reports as legal; this table itself never
    returns INFINITY (legality is the scheduler's business)."""
    def cost(block: int, mask: int, strategy: int) -> float:
        base = 0.05 + _u01(seed, block, mask, 0)
        if strategy == MERGE:
            return 0.05 + _u01(seed, block, mask, 1) * (1.0 / max(merge_frac, 1e-9))
        return base
    return cost


def integer_cost_table(times: Sequence[int]) -> Callable[[int, int, int], float]:
    """Additive costs L(S') = sum_{v in S'} t_v with integer t_v (exactly representable sums;
    SURVEY §8c "Additive => sequential")."""
    t = [int(v) for v in times]

    def cost(block: int, mask: int, strategy: int) -> float:
        s = 0
        i = 0
        m = mask
        while m:
            if m & 1:
                s += t[i]
            m >>= 1
            i += 1
        return float(s)
    return cost
