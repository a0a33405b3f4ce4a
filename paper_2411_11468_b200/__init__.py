"""paper_2411_11468_b200 — B200-native ν-LPA (arXiv 2411.11468) label-propagation hot path.

The product is the CUDA library ``libnulpa.so`` (sm_100a kernels behind the C ABI in
include/nulpa/nulpa.h) plus a C++ drop-in for ``labelprop::lpa``; this package is the
Python host mirror of the reference's engine interface over that ABI.
"""
from .labelprop import (CsrGraph, DegreePartition, DeviceGraph, EdgeList, ExecMode, FileFormat,
                        FormatError, build_csr, load_graph, InternalError,
                        LpaConfig, LpaResult, ProbeStrategy, RunStats, Tuning, ValidationError,
                        ValuePrecision, community_count, cross_check, lpa, modularity,
                        partition_by_degree, sync_step)

__all__ = [
    "CsrGraph", "DegreePartition", "DeviceGraph", "ExecMode", "InternalError", "LpaConfig",
    "LpaResult", "ProbeStrategy", "RunStats", "Tuning", "ValidationError", "ValuePrecision",
    "community_count", "cross_check", "lpa", "modularity", "partition_by_degree", "sync_step",
]
