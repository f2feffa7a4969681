"""tec-sm100: B200-native backend for the fused conv2d / depthwise_conv2d
operator path of the reference tec (arXiv 1802.04799 re-creation).

Public API (mirrors the reference, see ops.py):
    eval_operator, eval_graph_node, fused_conv, GraphNode
The compute runs in libtec_sm100.so (sm_100a kernels behind the C ABI of
include/tec_sm100.h); there is no CPU fallback.
"""
from ._abi import TecError, load  # noqa: F401
from .ops import (GraphNode, conv_desc, eval_graph_node,  # noqa: F401
                  eval_operator, fused_conv)

__all__ = ["TecError", "GraphNode", "eval_operator", "eval_graph_node",
           "fused_conv", "conv_desc", "load"]
