"""bench.py contract checks that run without a GPU: the reference arm (the CPU oracle, the tier's
reference) prints one JSON line with the contract's keys; the roofline accounting is consistent."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_contract_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--net", "fig2",
                          "--steps", "1", "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["higher_is_better"] is False
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["value"] > 0


def test_stage_roofline_accounting():
    """Per-stage roofline bytes/FLOPs on the Fig. 2 block: F counts unpadded MACs x 2,
    B counts each distinct stage input once, weights and outputs; an elided concat costs 0."""
    sys.path.insert(0, ROOT)
    import workloads as W
    from bench import stage_roofline
    from paper_2011_01302_b200 import Graph
    net = W.fig2_block()
    g = Graph.from_netspec(net)
    q = g.schedule([([1, 3, 4], 0), ([2], 0), ([5], 0)])
    peaks = {"hbm_gbs": 1000.0, "bf16_tflops": 1000.0, "tf32_tflops": 500.0}
    rows = stage_roofline(g, net, q, peaks)
    hw = 28 * 28
    f0 = 2 * hw * (128 * 64 * 9 + 64 * 64 + 96 * 64 * 9)
    assert rows[0]["flops"] == f0
    b0 = (64 * hw + 128 * 64 * 9 + 64 * 64 + 96 * 64 * 9 + (128 + 64 + 96) * hw) * 4   # x read once
    assert rows[0]["bytes"] == b0
    assert rows[2]["flops"] == 0 and rows[2]["bytes"] == 0                               # elided concat


def test_gpus_flag_relaunches_one_rank_per_gpu():
    """`bench.py --gpus 2` outside torchrun re-executes itself under torch.distributed.run (one
    process per GPU); exercised here on the reference arm, where rank 0 alone prints the line."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--net", "fig2",
                          "--gpus", "2", "--steps", "1", "--warmup", "3"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2
