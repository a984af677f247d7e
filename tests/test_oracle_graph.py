"""Pins for oracle/graph.py (O1 on whole networks, O2 schedule execution, merge, groups)."""
import json
import os

import numpy as np
import pytest
import torch

import workloads as W
from oracle import OracleGraph, scheduler as S
from oracle.graph import CONCURRENT, MERGE, ScheduleError

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ----------------------------------------------------------------------------- merge

def _merge_exact(net, ops):
    g = OracleGraph(net)
    vals = g.run_sequential(net.make_input())
    merged = g.run_merged(ops, vals)
    for i in ops:
        # padded taps add exact zeros and the non-zero terms keep their order: equal up to the sign of 0
        assert np.all(merged[i] == vals[i]), (net.name, i)


def test_merge_fig2_acd_and_pairs_exact():
    net = W.fig2_block()
    for ops in ([1, 3, 4], [1, 3], [1, 4], [3, 4]):
        _merge_exact(net, ops)


def test_merge_paper_example_128_plus_256_3x3():
    """Conv[a] 128 3x3 + Conv[b] 256 3x3 -> Merged Conv[a&b] with 384 3x3 kernels."""
    nb = W.netspec.NetBuilder("p192", (1, 32, 9, 9), 3)
    nb.conv(0, 128, 3, 1, 1)
    nb.conv(0, 256, 3, 1, 1)
    g = OracleGraph(nb.net)
    wm, bm, box, pad, splits = g.merged_conv([1, 2])
    assert wm.shape == (384, 32, 3, 3) and box == (3, 3) and pad == (1, 1) and splits == [(0, 128), (128, 384)]
    _merge_exact(nb.net, [1, 2])


def test_merge_1x3_3x1_becomes_3x3():
    """kernels 3x1 and 1x3 are expanded to 3x3 by padding zeros."""
    nb = W.netspec.NetBuilder("p571", (1, 16, 8, 8), 4)
    nb.conv(0, 24, (1, 3), 1, (0, 1))
    nb.conv(0, 8, (3, 1), 1, (1, 0))
    nb.conv(0, 16, 1, 1, 0)
    g = OracleGraph(nb.net)
    wm, _, box, pad, _ = g.merged_conv([1, 2, 3])
    assert box == (3, 3) and pad == (1, 1)
    assert np.all(wm[:24, :, 0, :] == 0) and np.all(wm[:24, :, 2, :] == 0)       # 1x3 sits in the middle row
    assert np.all(wm[24:32, :, :, 0] == 0) and np.all(wm[24:32, :, :, 2] == 0)   # 3x1 in the middle column
    assert np.all(wm[32:, :, 1, 1] == nb.net.ops[2].weight[:, :, 0, 0])           # 1x1 at the centre
    _merge_exact(nb.net, [1, 2, 3])


def test_merge_legality_reading_z4():
    net = W.fig2_block()
    g = OracleGraph(net)
    assert g.mergeable([1, 3, 4])
    assert not g.mergeable([1])            # |S'| >= 2
    assert not g.mergeable([1, 2])         # b reads a, not the shared input
    assert not g.mergeable([2, 3])
    net2 = W.tiny_mixed_net()
    g2 = OracleGraph(net2)
    ids = {o.name: i for i, o in enumerate(net2.ops, start=1)}
    assert g2.mergeable([ids["b1"], ids["b5_1"]])
    assert not g2.mergeable([ids["b1"], ids["pool"]])      # different type
    assert not g2.mergeable([ids["sep3"], ids["avg_excl"]])


# ----------------------------------------------------------------------------- groups / endings

def test_groups_fig3_example():
    """Fig. 3: stage {c, d, e} with edge c -> d -> groups {c, d} and {e}."""
    nb = W.netspec.NetBuilder("fig3", (1, 8, 4, 4), 1)
    a = nb.conv(0, 8, 1)           # a
    b = nb.conv(0, 8, 1)           # b
    c = nb.conv(a, 8, 1)           # c
    nb.conv(c, 8, 1)               # d
    nb.linear(nb.gavgpool(b), 8)   # e (matmul) on pooled b
    g = OracleGraph(nb.net)
    # local indices: a0 b1 c2 d3 gap4 e5; stage {c, d, e}
    assert g.groups(0, (1 << 2) | (1 << 3) | (1 << 5)) == [[2, 3], [5]]


def test_fig4_not_an_ending():
    """Fig. 4: S' containing d but not its successor g is not an ending."""
    preds = [[], [], [0], [1], [2], [3], [3]]    # a b c d e f g with d -> g
    net = W.dag_net(preds)
    g = OracleGraph(net)
    d, gg = 3, 6
    full = (1 << 7) - 1
    assert not S.is_ending(g.succ[0], full, 1 << d)
    assert S.is_ending(g.succ[0], full, (1 << d) | (1 << gg) | (1 << 5))


# ----------------------------------------------------------------------------- schedule execution

def test_every_fig2_schedule_equals_sequential_exactly():
    """O2 invariant: any valid Q gives the sequential outputs; merge stages build the
    merged kernel explicitly. Covers all 44 concurrent-only schedules plus every merge variant."""
    net = W.fig2_block()
    g = OracleGraph(net)
    x = net.make_input()
    ref = g.run_sequential(x)
    mem = g.block_members[0]
    n_sched = 0
    n_merge = 0
    for q in S.all_schedules(g.succ[0], g.pred[0], lambda m: g.mergeable(g.block_mask_ops(0, m))):
        qq = [([mem[i] for i in range(4) if (m >> i) & 1], t) for m, t in q] + [([5], CONCURRENT)]
        out = g.run_schedule(qq, x, np.random.default_rng(n_sched))
        for i in range(1, 6):
            assert np.all(out[i] == ref[i])
        n_sched += 1
        n_merge += any(t == MERGE for _, t in q)
    assert n_sched - n_merge == 44
    assert n_merge > 0


def test_validate_schedule_rejects_bad_orders():
    net = W.fig2_block()
    g = OracleGraph(net)
    with pytest.raises(ScheduleError):
        g.validate_schedule([([2], 0), ([1], 0), ([3], 0), ([4], 0), ([5], 0)])    # b before a
    with pytest.raises(ScheduleError):
        g.validate_schedule([([1, 2], MERGE), ([3], 0), ([4], 0), ([5], 0)])      # a->b cannot merge
    with pytest.raises(ScheduleError):
        g.validate_schedule([([1], 0), ([3], 0), ([4], 0), ([5], 0)])             # b missing
    g.validate_schedule([([1, 2, 3, 4], 0), ([5], 0)])                            # chain in one group


# ----------------------------------------------------------------------------- whole networks vs torchvision

def _bn_identity(bn, bias):
    bn.weight.data.fill_(1.0)
    bn.bias.data.copy_(torch.from_numpy(bias.astype(np.float64)))
    bn.running_mean.zero_()
    bn.running_var.fill_(1.0 - bn.eps)


@pytest.mark.slow
def test_inception_v3_topology_matches_torchvision_f64():
    """The whole Inception V3 oracle forward vs torchvision's module (BN set to identity + our bias)."""
    import torchvision
    net = W.inception_v3()
    m = torchvision.models.inception_v3(weights=None, aux_logits=False, init_weights=False).double().eval()
    mods = dict(m.named_modules())
    for o in net.ops:
        if o.kind == "conv":
            tv = o.name
            if "." in tv:
                pre, suf = tv.split(".")
                tv = pre + "." + ("branch_pool" if suf == "bpool" else "branch" + suf[1:])
            mod = mods[tv]
            mod.conv.weight.data.copy_(torch.from_numpy(o.weight.astype(np.float64)))
            _bn_identity(mod.bn, o.bias)
        elif o.kind == "linear":
            m.fc.weight.data.copy_(torch.from_numpy(o.weight.astype(np.float64)))
            m.fc.bias.data.copy_(torch.from_numpy(o.bias.astype(np.float64)))
    x = net.make_input()
    g = OracleGraph(net)
    y = g.run_sequential(x)[g.n][:, :, 0, 0]
    with torch.no_grad():
        ref = m(torch.from_numpy(x.astype(np.float64))).numpy()
    assert np.abs(y - ref).max() / np.abs(ref).max() < 1e-9


@pytest.mark.slow
def test_squeezenet_topology_matches_torchvision_f64():
    import torchvision
    net = W.squeezenet()
    m = torchvision.models.squeezenet1_0(weights=None).double().eval()
    fire_idx = {"fire2": 3, "fire3": 4, "fire4": 5, "fire5": 7, "fire6": 8, "fire7": 9, "fire8": 10, "fire9": 12}
    for o in net.ops:
        if o.kind != "conv":
            continue
        if o.name == "conv1":
            mod = m.features[0]
        elif o.name == "conv10":
            mod = m.classifier[1]
        else:
            fire, part = o.name.split(".")
            mod = getattr(m.features[fire_idx[fire]], part)
        mod.weight.data.copy_(torch.from_numpy(o.weight.astype(np.float64)))
        mod.bias.data.copy_(torch.from_numpy(o.bias.astype(np.float64)))
    x = net.make_input()
    g = OracleGraph(net)
    y = g.run_sequential(x)[g.n][:, :, 0, 0]
    with torch.no_grad():
        ref = m(torch.from_numpy(x.astype(np.float64))).numpy()
    assert np.abs(y - ref).max() / np.abs(ref).max() < 1e-12


def test_network_op_and_block_counts():
    """Table 2 reading, Z10: documented deviations are asserted here."""
    inc = OracleGraph(W.inception_v3())
    assert sum(o.kind == "conv" for o in inc.ops) == 94 and inc.shapes[inc.n] == (1, 1000, 1, 1)
    assert max(len(m) for m in inc.block_members.values()) == 12
    rw = OracleGraph(W.randwire_ws_small())
    assert max(len(m) for m in rw.block_members.values()) == 33          # Table 1: n = 33
    sq = OracleGraph(W.squeezenet())
    assert sq.shapes[sq.n] == (1, 1000, 1, 1)
