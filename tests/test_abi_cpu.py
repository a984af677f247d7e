"""CPU tests of the C-ABI library (no GPU): it loads, exports every symbol include/ios.h declares,
builds graphs with the oracle's shapes, rejects invalid input, and its DP — driven by a fixed cost
table through the ios_cost_fn callback — returns schedules bit-exact to the oracle's."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

import workloads as W
from oracle import OracleGraph, scheduler as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ios():
    import paper_2011_01302_b200 as pkg
    return pkg


def test_library_exports_every_declared_symbol(ios):
    hdr = open(os.path.join(ROOT, "include", "ios.h")).read()
    names = set(re.findall(r"\b(ios_[a-z_0-9]+)\s*\(", hdr))
    names -= {"ios_cost_fn"}
    lib = ctypes.CDLL(ios.LIB_PATH)
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    assert len(names) >= 24


@pytest.mark.parametrize("name", ["fig2", "tiny_mixed", "inception_v3", "squeezenet", "nasnet_a_large",
                                  "randwire_ws_small"])
def test_shapes_match_oracle(ios, name):
    net = W.build(name)
    g = ios.Graph.from_netspec(net)
    og = OracleGraph(net)
    assert g.num_ops == og.n
    for i in range(og.n + 1):
        assert g.op_shape(i) == og.shapes[i], (name, i)
    blocks = g.blocks()
    assert [b for b, _ in blocks] == og.block_ids
    assert [ops for _, ops in blocks] == [og.block_members[b] for b in og.block_ids]


def test_mergeable_matches_oracle(ios):
    net = W.inception_v3()
    g = ios.Graph.from_netspec(net)
    og = OracleGraph(net)
    rng = np.random.default_rng(0)
    for b in og.block_ids:
        mem = og.block_members[b]
        for _ in range(30):
            k = int(rng.integers(1, min(4, len(mem)) + 1))
            ops = sorted(rng.choice(mem, k, replace=False).tolist())
            assert g.mergeable(ops) == og.mergeable(ops), ops


def test_error_codes(ios):
    g = ios.Graph(1, 8, 8, 8)
    with pytest.raises(ios.IOSError) as e:
        ios.ios_add_op(g.handle, "conv", [5], 0, 8, (1, 1), weight=np.zeros(64, np.float32))
    assert e.value.status == 2                                     # dangling input
    a = ios.ios_add_op(g.handle, "conv", [0], 0, 8, (3, 3), pad=(1, 1), weight=np.zeros(8 * 8 * 9, np.float32))
    p = ios.ios_add_op(g.handle, "maxpool", [a], 0, kernel=(3, 3), stride=(2, 2))
    with pytest.raises(ios.IOSError) as e:
        ios.ios_add_op(g.handle, "add", [a, p], 0)
    assert e.value.status == 3                                     # add of 8x8 and 3x3 inputs
    with pytest.raises(ios.IOSError) as e:
        ios.ios_add_op(g.handle, "concat", [a, p], 0)
    assert e.value.status == 3
    ios.ios_add_op(g.handle, "maxpool", [a], 1, kernel=(3, 3), stride=(2, 2))
    with pytest.raises(ios.IOSError) as e:
        ios.ios_add_op(g.handle, "conv", [a], 0, 8, (1, 1), weight=np.zeros(64, np.float32))
    assert e.value.status == 4                                     # block 0 reopened
    with pytest.raises(ios.IOSError) as e:
        g.schedule([([3], 0), ([1], 0), ([2], 0)])
    assert e.value.status in (6, 7)
    with pytest.raises(ios.IOSError) as e:
        g.schedule([([1], 1), ([2], 0), ([3], 0)])
    assert e.value.status == 5                                     # merge of one op


def _lib_dp(g, cost, r, s, strategies="both"):
    q = g.schedule_dp(r, s, cost, strategies)
    return q.cost, [(st[0], st[1]) for st in q.stages], q.stats


@pytest.mark.parametrize("seed", range(30))
def test_dp_bit_exact_vs_oracle_random_dags(ios, seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(1, 11))
    net = W.dag_net(W.random_dag(n, float(rng.uniform(0.1, 0.6)), seed), conv_k=int(rng.choice([1, 3])))
    og = OracleGraph(net)
    g = ios.Graph.from_netspec(net)
    cost = W.random_cost_table(seed)
    r, s = [(None, None), (1, 8), (2, 3), (3, 8), (1, 1)][seed % 5]
    c_lib, q_lib, _ = _lib_dp(g, cost, r or 0, s or 0)
    c_or, q_or = S.dp(og, cost, r, s)
    assert c_lib == c_or
    assert q_lib == [(sorted(o), t) for o, t in q_or]


@pytest.mark.parametrize("name", ["fig2", "fig5", "inception_v3", "squeezenet", "tiny_mixed"])
@pytest.mark.parametrize("strategies", ["both", "merge", "parallel"])
def test_dp_bit_exact_vs_oracle_networks(ios, name, strategies):
    net = W.build(name)
    og = OracleGraph(net)
    g = ios.Graph.from_netspec(net)
    cost = W.random_cost_table(17)
    sset = {"both": S.BOTH, "merge": S.MERGE_ONLY, "parallel": S.PARALLEL_ONLY}[strategies]
    c_lib, q_lib, stats = _lib_dp(g, cost, 3, 8, strategies)
    c_or, q_or = S.dp(og, cost, 3, 8, sset)
    assert c_lib == c_or
    assert q_lib == [(sorted(o), t) for o, t in q_or]


def test_dp_stats_match_oracle_counts(ios):
    """ios_schedule_dp_ex's (states, transitions) equal the oracle's Fig. 5 / Table 1-style counts."""
    for name, r, s in [("fig5", 0, 0), ("fig2", 0, 0), ("inception_v3", 3, 8)]:
        net = W.build(name)
        og = OracleGraph(net)
        g = ios.Graph.from_netspec(net)
        _, _, (states, trans, _) = _lib_dp(g, W.random_cost_table(1), r, s)
        tot_states = tot_trans = 0
        for b in og.block_ids:
            st, tr, _ = S.count(og.succ[b], og.pred[b], r or None, s or None)
            tot_states += st
            tot_trans += tr
        assert (states, trans) == (tot_states, tot_trans), name


def test_additive_costs_sequential(ios):
    net = W.inception_v3()
    g = ios.Graph.from_netspec(net)
    c, q, _ = _lib_dp(g, lambda b, m, t: float(bin(m).count("1")), 3, 8)
    assert [o for o, _ in q] == [[i] for i in range(1, net.n_ops + 1)]
    assert c == float(net.n_ops)


def test_sequential_and_greedy_match_oracle(ios):
    for name in ["fig2", "inception_v3", "randwire_ws_small"]:
        net = W.build(name)
        og = OracleGraph(net)
        g = ios.Graph.from_netspec(net)
        assert [st[0] for st in g.schedule_sequential().stages] == [o for o, _ in S.sequential(og)]
        assert [st[0] for st in g.schedule_greedy().stages] == [sorted(o) for o, _ in S.greedy(og)]


def test_schedule_roundtrip_and_validation(ios):
    net = W.fig2_block()
    g = ios.Graph.from_netspec(net)
    q = g.schedule([([1, 3, 4], 1), ([2], 0), ([5], 0)])
    assert [(o, t) for o, t, _ in q.stages] == [([1, 3, 4], 1), ([2], 0), ([5], 0)]
    g.schedule([([1, 2, 3, 4], 0), ([5], 0)])                    # chain a->b inside one group
    with pytest.raises(Exception):
        g.schedule([([1, 2], 1), ([3], 0), ([4], 0), ([5], 0)])  # a->b cannot merge


def test_latency_cache_roundtrip(ios, tmp_path):
    net = W.fig2_block()
    g = ios.Graph.from_netspec(net)
    p = str(tmp_path / "cache.txt")
    g.save_latency_cache(p)
    g.load_latency_cache(p)
    g2 = ios.Graph.from_netspec(W.fig5_graph())
    with pytest.raises(ios.IOSError):
        g2.load_latency_cache(p)


def test_no_cpu_fallback_without_gpu(ios):
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    net = W.fig2_block()
    g = ios.Graph.from_netspec(net)
    with pytest.raises(ios.IOSError) as e:
        g.stage_latency([1])
    assert e.value.status == 8                                     # IOS_ERR_CUDA, never a CPU path


def test_loaded_library_is_built_from_these_sources(ios):
    """Provenance: the .so the tests load carries the content hash of the sources in this tree
    (build.py compiles it in as ios_build_id()), so a stale or foreign binary cannot pass for HEAD."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("_ios_build", os.path.join(ROOT, "paper_2011_01302_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    assert ios.ios.ios_build_id() == mod.source_hash()


@pytest.mark.timeout(60)
@pytest.mark.parametrize("bad", [math.inf, math.nan])
def test_dp_all_infinite_costs_is_an_error_not_a_hang(ios, bad):
    """Every ending costing inf/NaN leaves no finite schedule: the library reports it (the oracle
    raises too) instead of looping in Algorithm 1's L8-11 reconstruction."""
    g = ios.Graph.from_netspec(W.fig2_block())
    with pytest.raises(ios.IOSError) as e:
        g.schedule_dp(3, 8, lambda b, m, t: bad)
    assert e.value.status == 11


def test_latency_cache_keeps_entries_after_an_infinite_one(ios, tmp_path):
    """An unsupported stage is cached as inf; it must round-trip and must not truncate the load."""
    g = ios.Graph.from_netspec(W.fig2_block())
    p = tmp_path / "cache.txt"
    g.save_latency_cache(str(p))
    sig = p.read_text().splitlines()[0]
    p.write_text(sig + "\n7 1 0 inf\n7 2 0 0.0125\n7 13 1 0.03\n")
    g.load_latency_cache(str(p))
    p2 = tmp_path / "cache2.txt"
    g.save_latency_cache(str(p2))
    rows = sorted(l.split() for l in p2.read_text().splitlines()[1:])
    assert rows == [["7", "1", "0", "inf"], ["7", "13", "1", "0.029999999999999999"], ["7", "2", "0", "0.012500000000000001"]]
    p.write_text(sig + "\n7 1 0 abc\n")
    with pytest.raises(ios.IOSError):
        g.load_latency_cache(str(p))
