"""Pins for oracle/scheduler.py (Algorithm 1) against the paper's worked examples,
closed forms and brute force."""
import json
import math
import os

import numpy as np
import pytest

import workloads as W
from oracle import OracleGraph, scheduler as S

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def _block(net, b=0):
    g = OracleGraph(net)
    return g, g.succ[b], g.pred[b]


def test_fig5_states_transitions_schedules():
    gold = _load("fig5_dp_counts.json")
    g, succ, pred = _block(W.fig5_graph())
    assert S.count(succ, pred) == (gold["states"], gold["transitions"], gold["schedules"])
    names = gold["graph"]["ops"]
    got = [[names[i] for i in range(3) if (m >> i) & 1] for m in S.endings(succ, pred, 0b111)]
    assert sorted(map(tuple, got)) == sorted(map(tuple, gold["endings_of_V"]))


def test_fig2_counts_and_greedy():
    gold = _load("fig2_greedy.json")
    net = W.fig2_block()
    g, succ, pred = _block(net)
    sp = gold["dp_space"]
    assert S.count(succ, pred) == (sp["states"], sp["transitions"], sp["schedules_concurrent_only"])
    names = {o.name: i for i, o in enumerate(net.ops, start=1)}
    want = [[names[n] for n in st] for st in gold["greedy_block0"]]
    got = [sorted(ops) for ops, _ in S.greedy(g) if g.local[ops[0]][0] == 0]
    assert got == [sorted(s) for s in want]


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6])
def test_chain_closed_forms(n):
    preds = [[]] + [[i - 1] for i in range(1, n)]
    _, succ, pred = _block(W.dag_net(preds))
    states, trans, sched = S.count(succ, pred)
    assert (states, trans, sched) == (n + 1, n * (n + 1) // 2, 2 ** (n - 1))


def test_appendix_tight_example_counts():
    """Lemma 3 / Fig. 13: d chains of c ops; non-empty transitions = C(c+2,2)^d - (c+1)^d."""
    for case in _load("appendix_tight.json")["cases"]:
        c, d = case["c"], case["d"]
        preds = []
        for chain in range(d):
            for j in range(c):
                preds.append([len(preds) - 1] if j > 0 else [])
        _, succ, pred = _block(W.dag_net(preds))
        states, trans, _ = S.count(succ, pred)
        assert math.comb(c + 2, 2) ** d == case["pairs_with_empty"]
        assert trans == case["transitions"] == case["pairs_with_empty"] - (c + 1) ** d
        assert states == (c + 1) ** d


def test_table1_bound_column():
    """C(n/d + 2, 2)^d with fractional n/d reproduces Table 1's bound column."""
    for row in _load("table1_bounds.json")["rows"]:
        x = row["n"] / row["d"]
        bound = ((x + 2) * (x + 1) / 2) ** row["d"]
        assert float(f"{bound:.1e}") == pytest.approx(row["bound"], rel=1e-9), row


def _dp_vs_brute(net, seed, r=None, s=None, strategies=S.BOTH):
    g, succ, pred = _block(net)
    cost = W.random_cost_table(seed)
    merge = lambda m: g.mergeable(g.block_mask_ops(0, m))
    bdp = S.BlockDP(succ, pred, lambda m, t: cost(0, m, t), merge, r, s, strategies)
    c_dp, q = bdp.run()
    c_bf, _ = S.brute_force(succ, pred, lambda m, t: cost(0, m, t), merge, r, s)
    return c_dp, c_bf, q


@pytest.mark.parametrize("seed", range(40))
def test_dp_equals_brute_force_bit_exact(seed):
    """DP cost == brute-force minimum over all schedules, bit-exactly (SURVEY §8c pin)."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 7))
    preds = W.random_dag(n, float(rng.uniform(0.1, 0.7)), seed)
    net = W.dag_net(preds, conv_k=int(rng.choice([1, 3])))
    rs = [(None, None), (1, 2), (2, 3), (3, 8)][seed % 4]
    c_dp, c_bf, q = _dp_vs_brute(net, seed, *rs)
    assert c_dp == c_bf
    # the returned Q really costs c_dp when summed left to right
    cost = W.random_cost_table(seed)
    tot = 0.0
    for m, t in q:
        tot = tot + cost(0, m, t)
    assert tot == c_dp


@pytest.mark.parametrize("seed", range(20))
def test_additive_costs_give_sequential(seed):
    """If L(S') = sum t_v with integer t_v every schedule ties and canonical order (Z1) returns the
    insertion-order sequential schedule."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(1, 9))
    net = W.dag_net(W.random_dag(n, 0.4, seed))
    g, succ, pred = _block(net)
    cost = W.integer_cost_table(rng.integers(1, 50, n))
    bdp = S.BlockDP(succ, pred, lambda m, t: cost(0, m, t), lambda m: g.mergeable(g.block_mask_ops(0, m)), 3, 8)
    _, q = bdp.run()
    assert [m for m, _ in q] == [1 << i for i in range(n)]


def test_strategy_tie_goes_to_merge():
    """Alg. 1 L30 uses strict <: L_concurrent == L_merge returns operator merge (Z2)."""
    net = W.fig2_block()
    g, succ, pred = _block(net)
    bdp = S.BlockDP(succ, pred, lambda m, t: 1.0, lambda m: g.mergeable(g.block_mask_ops(0, m)))
    assert bdp.generate_stage(0b1101) == (1.0, S.MERGE)       # {a, c, d}
    assert bdp.generate_stage(0b0011) == (1.0, S.CONCURRENT)  # {a, b}: not mergeable


@pytest.mark.parametrize("seed", range(10))
def test_dominance_and_pruning_monotonicity(seed):
    rng = np.random.default_rng(200 + seed)
    n = int(rng.integers(3, 9))
    net = W.dag_net(W.random_dag(n, 0.3, seed))
    g, succ, pred = _block(net)
    cost = W.random_cost_table(seed)
    merge = lambda m: g.mergeable(g.block_mask_ops(0, m))
    f = lambda m, t: cost(0, m, t)
    seq = 0.0
    for i in range(n):
        seq = seq + f(1 << i, S.CONCURRENT)
    gq = [m for m in S.greedy(g)]
    gr = 0.0
    for ops, _ in gq:
        mask = sum(1 << g.local[v][1] for v in ops)
        gr = gr + min(f(mask, S.CONCURRENT), f(mask, S.MERGE) if merge(mask) else math.inf)
    full, _ = S.BlockDP(succ, pred, f, merge).run()
    assert full <= seq and full <= gr
    prev = math.inf
    for r, s in [(1, 1), (1, 3), (2, 3), (3, 8), (None, None)]:
        c, _ = S.BlockDP(succ, pred, f, merge, r, s).run()
        assert c <= seq and c <= prev
        prev = c


def test_ios_merge_and_parallel_variants():
    """IOS-Merge / IOS-Parallel: Parallel never merges; Merge never runs a multi-op
    concurrent stage; Both is no worse than either."""
    net = W.fig2_block()
    g, succ, pred = _block(net)
    cost = W.random_cost_table(7)
    merge = lambda m: g.mergeable(g.block_mask_ops(0, m))
    f = lambda m, t: cost(0, m, t)
    cb, _ = S.BlockDP(succ, pred, f, merge, strategies=S.BOTH).run()
    cp, qp = S.BlockDP(succ, pred, f, merge, strategies=S.PARALLEL_ONLY).run()
    cm, qm = S.BlockDP(succ, pred, f, merge, strategies=S.MERGE_ONLY).run()
    assert all(t == S.CONCURRENT for _, t in qp)
    assert all(t == S.MERGE or (m & (m - 1)) == 0 for m, t in qm)
    assert cb <= cp and cb <= cm


def test_whole_graph_dp_concatenates_blocks():
    net = W.inception_v3()
    g = OracleGraph(net)
    cost = W.integer_cost_table([1] * 64)
    total, q = S.dp(g, cost, 3, 8)
    assert [v for ops, _ in q for v in ops] == list(range(1, g.n + 1))
    assert total == g.n
    g.validate_schedule(q)
