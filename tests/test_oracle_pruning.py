"""Pins for the oracle's schedule pruning P(r, s) (Sec. 4.3) and its brute force.

P(S, S') = True iff the ending S' has at most s groups and each group has at most r operators
(P:415-416); groups are connected components (Z3). These tests check the oracle's
counts against (1) hand-counted fixtures (tests/golden/pruning_counts.json) and (2) a closed form
derived from that definition for d independent chains of c ops, and check the DP against a brute
force written here from scratch (ordered set partitions, its own group count), sharing nothing with
oracle/scheduler.py's ending enumerator.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import workloads as W
from oracle import OracleGraph, scheduler as S

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "pruning_counts.json")


def chains(c: int, d: int):
    """succ/pred masks of d independent chains of c ops; op (chain i, position j) has index i*c + j."""
    n = c * d
    succ, pred = [0] * n, [0] * n
    for i in range(d):
        for j in range(c - 1):
            u, v = i * c + j, i * c + j + 1
            succ[u] |= 1 << v
            pred[v] |= 1 << u
    return succ, pred


def independent(n: int):
    return [0] * n, [0] * n


GRAPHS = {"chain of 3 ops": lambda: chains(3, 1), "2 independent chains of 2 ops": lambda: chains(2, 2),
          "3 independent ops": lambda: independent(3)}


@pytest.mark.parametrize("case", json.load(open(GOLD))["cases"], ids=lambda c: f"{c['graph']}-r{c['r']}-s{c['s']}")
def test_hand_counted_pruned_transitions(case):
    succ, pred = GRAPHS[case["graph"]]()
    _, trans, _ = S.count(succ, pred, case["r"], case["s"])
    assert trans == case["transitions"], case["why"]


def closed_form_transitions(c: int, d: int, r: int, s: int) -> int:
    """d independent chains of c ops. A state keeps a prefix of length l_i of chain i (endings peel
    suffixes); an ending takes a suffix of length k_i <= l_i of each chain, not all zero. A
    non-empty suffix of a chain is exactly ONE group of k_i ops, so P(r, s) admits it iff
    #{i: k_i > 0} <= s and every k_i <= r. Summing over the (c+1)^d states:
        T = sum_{j=1}^{min(s,d)} C(d, j) * A^j * (c+1)^(d-j),   A = sum_{l=0}^{c} min(l, r).
    Unpruned (r >= c, s >= d) this is C(c+2,2)^d - (c+1)^d, Appendix A's tight count."""
    A = sum(min(l, r) for l in range(c + 1))
    return sum(math.comb(d, j) * A ** j * (c + 1) ** (d - j) for j in range(1, min(s, d) + 1))


@pytest.mark.parametrize("c,d", [(1, 1), (3, 1), (5, 1), (2, 2), (3, 2), (2, 3), (4, 2), (1, 5), (3, 3)])
def test_pruned_transitions_closed_form(c, d):
    succ, pred = chains(c, d)
    for r in range(1, c + 2):
        for s in range(1, d + 2):
            states, trans, _ = S.count(succ, pred, r, s)
            assert states == (c + 1) ** d                 # singletons keep every state reachable (Z7)
            assert trans == closed_form_transitions(c, d, r, s), (c, d, r, s)
    assert closed_form_transitions(c, d, c, d) == math.comb(c + 2, 2) ** d - (c + 1) ** d


def test_chain_r1_gives_n_transitions():
    for n in range(1, 8):
        succ, pred = chains(n, 1)
        assert S.count(succ, pred, 1, 8)[1] == n


def test_survey_inception_e_counts():
    """SURVEY.md Appendix ('DP state-space facts', counted by a scratch script in the survey
    session, not by this oracle): the Inception-E block reading has 5040 transitions unpruned and
    4631 / 3571 / 1966 at (r, s) = (3, 8) / (2, 8) / (1, 8)."""
    og = OracleGraph(W.inception_v3())
    blk = [b for b in og.block_ids if any(og.ops[v - 1].name.startswith("Mixed_7b") for v in og.block_members[b])][0]
    succ, pred = og.succ[blk], og.pred[blk]
    assert S.count(succ, pred)[1] == 5040
    assert [S.count(succ, pred, r, 8)[1] for r in (3, 2, 1)] == [4631, 3571, 1966]


# ------------------------------------------------------------------ independent brute force
def _groups(succ, pred, members):
    """Number of connected components and the largest one, by union-find (not oracle.components)."""
    parent = {u: u for u in members}

    def find(u):
        while parent[u] != u:
            parent[u] = parent[parent[u]]
            u = parent[u]
        return u

    for u in members:
        for v in members:
            if (succ[u] >> v) & 1:
                parent[find(u)] = find(v)
    sizes = {}
    for u in members:
        sizes[find(u)] = sizes.get(find(u), 0) + 1
    return len(sizes), max(sizes.values())


def brute_min(succ, pred, cost, mergeable, r, s):
    """min over every ordered set partition (stage 0 first) that is a valid schedule: for every
    edge u -> v, stage(u) <= stage(v) (a same-stage edge lies inside one group); every stage
    passes P(r, s); each stage takes either legal strategy. Cost = left fold in execution order."""
    n = len(succ)
    best = math.inf
    for k in range(1, n + 1):
        for assign in itertools.product(range(k), repeat=n):
            if len(set(assign)) != k:
                continue
            if any((succ[u] >> v) & 1 and assign[u] > assign[v] for u in range(n) for v in range(n)):
                continue
            stages = [[u for u in range(n) if assign[u] == i] for i in range(k)]
            ok = True
            for st in stages:
                ng, big = _groups(succ, pred, st)
                if (s is not None and ng > s) or (r is not None and big > r):
                    ok = False
                    break
            if not ok:
                continue
            masks = [sum(1 << u for u in st) for st in stages]
            opts = [[cost(m, S.CONCURRENT)] + ([cost(m, S.MERGE)] if mergeable(m) else []) for m in masks]
            for choice in itertools.product(*opts):
                tot = 0.0
                for x in choice:
                    tot = tot + x
                best = min(best, tot)
    return best


@pytest.mark.parametrize("seed", range(12))
def test_dp_equals_independent_brute_force(seed):
    rng = np.random.default_rng(300 + seed)
    n = int(rng.integers(2, 6))
    net = W.dag_net(W.random_dag(n, float(rng.uniform(0.2, 0.6)), seed))
    og = OracleGraph(net)
    b = og.block_ids[0]
    succ, pred = og.succ[b], og.pred[b]
    table = W.random_cost_table(seed)
    cost = lambda m, t: table(b, m, t)
    merge = lambda m: og.mergeable(og.block_mask_ops(b, m))
    r, s = [(None, None), (1, 8), (2, 1), (1, 2), (3, 8), (2, 2)][seed % 6]
    c_dp, _ = S.BlockDP(succ, pred, cost, merge, r, s).run()
    assert c_dp == brute_min(succ, pred, cost, merge, r, s)
