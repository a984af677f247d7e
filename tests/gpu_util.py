"""Helpers for the -m gpu parity tests: run the CUDA path through the C-ABI and compare with the
oracle on the same seeded inputs (Z13 tolerance metric)."""
import numpy as np

from oracle import OracleGraph

TOL = {"tf32": 5e-3, "bf16": 2e-2}     # BASELINE.json north_star, normwise max relative error


def rel_err(y, ref) -> float:
    """Z13: max|y - ref| / max|ref| over one tensor."""
    y = np.asarray(y, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = np.abs(ref).max()
    if den == 0:
        return float(np.abs(y).max())
    return float(np.abs(y - ref).max() / den)


def per_op_errors(net, g, math, ops=None):
    """(ii) per op: the oracle is fed the GPU's own inputs of that op (read back through
    ios_op_output), so errors do not compound through depth."""
    og = OracleGraph(net)
    errs = {}
    cache = {}

    def gpu_val(u):
        if u not in cache:
            cache[u] = g.op_output(u).cpu().numpy().astype(np.float64)
        return cache[u]

    for i in (ops or range(1, og.n + 1)):
        o = og.ops[i - 1]
        vals = {u: gpu_val(u) for u in o.inputs}
        ref = og.run_op(i, vals)
        errs[i] = rel_err(gpu_val(i), ref)
    return errs
