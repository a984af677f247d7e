"""GPU parity: the CUDA stage executor (through the C-ABI) vs the oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star; metric DESIGN.md Z13): TF32 5e-3, BF16 2e-2 normwise, per op
(oracle fed the GPU's own inputs) and end to end.
"""
import numpy as np
import pytest

import workloads as W
from oracle import OracleGraph, scheduler as S
from tests.gpu_util import TOL, per_op_errors, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    return torch


def _run(net, math, schedule="sequential", torch=None, r=3, s=8):
    from paper_2011_01302_b200 import Graph
    g = Graph.from_netspec(net, math)
    if schedule == "sequential":
        q = g.schedule_sequential()
    elif schedule == "greedy":
        q = g.schedule_greedy()
    else:
        q = g.schedule(schedule)
    x = net.make_input()
    xt = torch.from_numpy(x).cuda()
    y = g.run(q, xt)
    torch.cuda.synchronize()
    return g, q, y.cpu().numpy()


@pytest.mark.parametrize("math", ["tf32", "bf16"])
def test_fig2_sequential_per_op_and_end_to_end(torch_cuda, math):
    net = W.fig2_block(math=math)
    g, q, y = _run(net, math, "sequential", torch_cuda)
    errs = per_op_errors(net, g, math)
    assert max(errs.values()) < TOL[math], errs
    ref = OracleGraph(net).run_sequential(net.make_input())[net.n_ops]
    assert rel_err(y, ref) < TOL[math]


@pytest.mark.parametrize("math", ["tf32", "bf16"])
def test_fig2_every_schedule(torch_cuda, math):
    """All 44 concurrent-only schedules of the Fig. 2 block plus every merge variant (one launch per
    stage; chains inside a stage use in-kernel dependency counters) match the oracle."""
    from paper_2011_01302_b200 import Graph
    net = W.fig2_block(math=math)
    og = OracleGraph(net)
    x = net.make_input()
    ref = og.run_sequential(x)[og.n]
    g = Graph.from_netspec(net, math)
    xt = torch_cuda.from_numpy(x).cuda()
    mem = og.block_members[0]
    n = 0
    for qq in S.all_schedules(og.succ[0], og.pred[0], lambda m: og.mergeable(og.block_mask_ops(0, m))):
        stages = [([mem[i] for i in range(4) if (m >> i) & 1], t) for m, t in qq] + [([5], 0)]
        q = g.schedule(stages)
        y = g.run(q, xt).cpu().numpy()
        assert rel_err(y, ref) < TOL[math], stages
        n += 1
    assert n >= 44


@pytest.mark.parametrize("math", ["tf32", "bf16"])
def test_tiny_mixed_all_op_kinds(torch_cuda, math):
    net = W.tiny_mixed_net(math=math)
    for sched in ("sequential", "greedy"):
        g, q, y = _run(net, math, sched, torch_cuda)
        errs = per_op_errors(net, g, math)
        assert max(errs.values()) < TOL[math], (sched, errs)
        ref = OracleGraph(net).run_sequential(net.make_input())[net.n_ops]
        assert rel_err(y, ref) < TOL[math]


def test_ios_stage_latency_positive(torch_cuda):
    from paper_2011_01302_b200 import Graph, MERGE
    net = W.fig2_block()
    g = Graph.from_netspec(net)
    t1 = g.stage_latency([1])
    t_all = g.stage_latency([1, 2, 3, 4])
    t_m = g.stage_latency([1, 3, 4], MERGE)
    assert 0 < t1 < 1.0 and 0 < t_all < 1.0 and 0 < t_m < 1.0


@pytest.mark.parametrize("name,math", [("inception_v3", "tf32"), ("squeezenet", "tf32"), ("randwire_ws_small", "bf16"),
                                       ("nasnet_a_large", "tf32")])
def test_network_sequential_and_greedy(torch_cuda, name, math):
    """Full networks at BASELINE.json's sizes: per-op parity (every op, oracle fed the GPU's inputs)
    under the sequential schedule, end-to-end parity under sequential and greedy."""
    net = W.build(name, math=math)
    x = net.make_input()
    ref = OracleGraph(net).run_sequential(x)[net.n_ops]
    g, q, y = _run(net, math, "sequential", torch_cuda)
    errs = per_op_errors(net, g, math)
    worst = max(errs, key=errs.get)
    assert errs[worst] < TOL[math], (worst, net.op(worst).name, errs[worst])
    assert rel_err(y, ref) < TOL[math]
    _, _, y2 = _run(net, math, "greedy", torch_cuda)
    assert rel_err(y2, ref) < TOL[math]


@pytest.mark.parametrize("name", ["fig2", "tiny_mixed"])
def test_fp32_simt_mode_1e5(torch_cuda, name):
    """IOS_MATH_FP32_SIMT: exact fp32 storage, CUDA-core FMA GEMM; north star tolerance 1e-5."""
    net = W.build(name)
    g, q, y = _run(net, "fp32_simt", "sequential", torch_cuda)
    errs = per_op_errors(net, g, "fp32_simt")
    assert max(errs.values()) < 1e-5, errs
    ref = OracleGraph(net).run_sequential(net.make_input())[net.n_ops]
    assert rel_err(y, ref) < 1e-5
    _, _, y2 = _run(net, "fp32_simt", "greedy", torch_cuda)
    assert rel_err(y2, ref) < 1e-5


@pytest.mark.parametrize("batch,hw,math", [(1, 37, "tf32"), (1, 37, "bf16"), (3, 7, "tf32"), (2, 9, "bf16"),
                                           (1, 150, "bf16")])
def test_conv_zoo_im2col_paths(torch_cuda, batch, hw, math):
    """Every conv shape class through the im2col paths (tap-TMA patches incl. multi-image and
    multi-column-tile patches, the cp.async gather, 1x1 TMA): per op under the sequential schedule,
    and the {3x3, 1x1, 5x5} group as one merged stage."""
    from paper_2011_01302_b200 import MERGE
    net = W.build("conv_zoo", batch=batch, hw=hw, math=math)
    g, q, y = _run(net, math, "sequential", torch_cuda)
    errs = per_op_errors(net, g, math)
    worst = max(errs, key=errs.get)
    assert errs[worst] < TOL[math], (worst, net.op(worst).name, errs[worst])
    stages = [([i], 0) for i in range(1, 12)] + [([12, 13, 14], MERGE), ([15], 0)]
    g.run(g.schedule(stages), torch_cuda.from_numpy(net.make_input()).cuda())
    torch_cuda.cuda.synchronize()
    errs = per_op_errors(net, g, math, ops=[12, 13, 14])
    assert max(errs.values()) < TOL[math], errs


@pytest.mark.parametrize("batch,hw,math", [(1, 37, "tf32"), (1, 37, "bf16"), (2, 7, "tf32"), (3, 9, "bf16"),
                                           (1, 150, "bf16"), (1, 83, "tf32")])
def test_sepconv_zoo_fused_depthwise(torch_cuda, batch, hw, math):
    """Fused Relu-SepConv (the depthwise half computed by the producer warps into the
    pointwise GEMM's A operand): every window / stride / aggregation / patch-geometry class, per op
    under the sequential schedule, then the whole block as ONE concurrent stage (the chain waits on
    an in-kernel counter)."""
    net = W.build("sepconv_zoo", batch=batch, hw=hw, math=math)
    ref = OracleGraph(net).run_sequential(net.make_input())[net.n_ops]
    g, q, y = _run(net, math, "sequential", torch_cuda)
    errs = per_op_errors(net, g, math)
    worst = max(errs, key=errs.get)
    assert errs[worst] < TOL[math], (worst, net.op(worst).name, errs[worst])
    assert rel_err(y, ref) < TOL[math]
    g2, _, y2 = _run(net, math, [(list(range(1, net.n_ops + 1)), 0)], torch_cuda)
    errs = per_op_errors(net, g2, math)
    worst = max(errs, key=errs.get)
    assert errs[worst] < TOL[math], (worst, net.op(worst).name, errs[worst])
    assert rel_err(y2, ref) < TOL[math]


def test_deterministic_split_k_slabs(torch_cuda):
    """IOS_SLAB_SPLITS=32: every split-K problem stores per-split slabs that the finalize sums in
    split order, so repeated runs are bitwise identical (SURVEY §5 determinism mode); parity holds.
    Runs in a subprocess because the library reads the knob once per process."""
    import os
    import subprocess
    import sys
    code = r'''
import hashlib, numpy as np, torch, workloads as W
from paper_2011_01302_b200 import Graph
net = W.build("conv_zoo", batch=1, hw=37, math="tf32")
g = Graph.from_netspec(net, "tf32")
q = g.schedule_sequential()
x = torch.from_numpy(net.make_input()).cuda()
hs = []
for _ in range(3):
    g.run(q, x); torch.cuda.synchronize()
    hs.append(hashlib.sha1(b"".join(g.op_output(i).cpu().numpy().tobytes() for i in range(1, net.n_ops + 1))).hexdigest())
print(len(set(hs)))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, IOS_SLAB_SPLITS="32", PYTHONPATH=root)
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip().splitlines()[-1] == "1", out.stdout


def test_tuned_schedule_parity(torch_cuda):
    """ios_schedule_tune re-tiles stages (split-K granularity) by measurement: the outputs still
    match the oracle per op, for the sequential and greedy schedules of the conv zoo."""
    from paper_2011_01302_b200 import Graph
    net = W.build("conv_zoo", batch=1, hw=37, math="tf32")
    g = Graph.from_netspec(net, "tf32")
    x = torch_cuda.from_numpy(net.make_input()).cuda()
    for q in (g.schedule_sequential(), g.schedule_greedy()):
        g.tune(q)
        g.run(q, x)
        torch_cuda.cuda.synchronize()
        errs = per_op_errors(net, g, "tf32")
        worst = max(errs, key=errs.get)
        assert errs[worst] < TOL["tf32"], (worst, net.op(worst).name, errs[worst])
