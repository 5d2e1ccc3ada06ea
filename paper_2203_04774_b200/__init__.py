"""trigpu: B200-native (sm_100a) triangle listing over order-oriented DAGs.

Drop-in for the listing path of the reference ``trilist`` library
(arXiv 2203.04774): OrientedView construction + list_app / list_apm + sinks,
as hand-written CUDA kernels behind the C-ABI in ``include/trigpu.h``.
"""
from .engine import (APM, APP, ChecksumSink, CollectingSink, CompositeSink, Context,
                     CountingSink, ListingStats, OrientedView, TrigpuError, VertexCountSink,
                     default_context, list_app, list_app_parallel, list_apm, list_apm_parallel,
                     orient)
from .host import (ORDERINGS, CostReport, Graph, Ordering, check_order, compute_order, core_order,
                   cost_report, degree_order, gen_chung_lu, gen_gnm, gen_rmat, gen_ws,
                   identity_order, neigh_order, random_order, split_order)

__all__ = [
    "APM", "APP", "ChecksumSink", "CollectingSink", "CompositeSink", "Context", "CountingSink",
    "ListingStats", "OrientedView", "TrigpuError", "VertexCountSink", "default_context",
    "list_app", "list_app_parallel", "list_apm", "list_apm_parallel", "orient", "ORDERINGS",
    "CostReport", "Graph", "Ordering", "check_order", "compute_order", "core_order",
    "cost_report", "degree_order", "gen_chung_lu", "gen_gnm", "gen_rmat", "gen_ws",
    "identity_order", "neigh_order", "random_order", "split_order",
]
