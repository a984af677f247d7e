"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package is the ONLY code both sides see. It generates graph descriptions (topology,
hyper-parameters, seeded weights), input tensors and cost tables. It contains none of the
method's arithmetic: no convolution, pooling, shape inference, DP or scheduling.
See DESIGN.md "Input recipe".
"""
from .netspec import NetSpec, OpSpec, OP_KINDS, bf16_round
from .networks import (fig2_block, fig5_graph, inception_v3, squeezenet, nasnet_a_large,
                       randwire_ws_small, build, NETWORKS, tiny_mixed_net)
from .randdag import random_dag, dag_net, random_cost_table, integer_cost_table, CONCURRENT, MERGE

__all__ = ["NetSpec", "OpSpec", "OP_KINDS", "bf16_round", "fig2_block", "fig5_graph",
           "inception_v3", "squeezenet", "nasnet_a_large", "randwire_ws_small", "build",
           "NETWORKS", "tiny_mixed_net", "random_dag", "dag_net", "CONCURRENT", "MERGE", "random_cost_table", "integer_cost_table"]
