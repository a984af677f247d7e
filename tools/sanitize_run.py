"""Small runs of the stage executor for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): the Fig. 2 block under a merge + chain schedule, the conv zoo (every im2col path,
split-K) and the sepconv zoo (fused depthwise producers) as one concurrent stage each.

  compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2011_01302_b200 import Graph, MERGE  # noqa: E402

runs = [("fig2", {}, [([1, 3, 4], MERGE), ([2], 0), ([5], 0)]),
        ("fig2", {}, [([1, 2, 3, 4], 0), ([5], 0)]),
        ("conv_zoo", dict(batch=1, hw=19), None),
        ("sepconv_zoo", dict(batch=1, hw=19), "one")]
for name, kw, stages in runs:
    net = W.build(name, **kw)
    g = Graph.from_netspec(net, "tf32")
    if stages is None:
        q = g.schedule_sequential()
    elif stages == "one":
        q = g.schedule([(list(range(1, net.n_ops + 1)), 0)])
    else:
        q = g.schedule(stages)
    x = torch.from_numpy(net.make_input()).cuda()
    for _ in range(2):
        g.run(q, x)
    g.sync()
    print(name, "ok", flush=True)
