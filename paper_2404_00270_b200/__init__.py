"""B200-native WBPR: vertex-centric push-relabel max-flow / min-cut on sm_100a.

The product is the C-ABI library ``libwbpr.so`` (include/wbpr.h) built from
``csrc/`` by ``build.py``; ``wbpr`` is its thin ctypes binding.
"""
from .wbpr import (WbprError, Workspace, barrier_cost, bipartite_match, build_residual, load, maxflow,
                   maxflow_batch, options, residual, trace, version, workspace_size)

__all__ = ["WbprError", "Workspace", "barrier_cost", "bipartite_match", "build_residual", "load", "maxflow",
           "maxflow_batch", "options", "residual", "trace", "version", "workspace_size"]
