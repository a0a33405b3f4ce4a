"""ctypes binding of the nulpa C ABI (include/nulpa/nulpa.h).

The shared library is built in-tree by ``python -m paper_2411_11468_b200.build``.
There is no fallback: if libnulpa.so is missing or no CUDA device is usable, the
calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libnulpa.so"

NULPA_OK, NULPA_EINVAL, NULPA_ENOMEM, NULPA_EINTERNAL, NULPA_ECUDA, NULPA_EOTHER, NULPA_EFORMAT = range(7)
NULPA_FORMAT_MATRIX_MARKET, NULPA_FORMAT_EDGE_LIST = 0, 1
NULPA_LAYOUT_IDENTITY, NULPA_LAYOUT_DEGREE_BUCKETS = 0, 1


class nulpa_csr(C.Structure):
    _fields_ = [("n", C.c_uint32), ("reserved", C.c_uint32), ("m2", C.c_uint64),
                ("offsets", C.c_void_p), ("targets", C.c_void_p), ("weights", C.c_void_p)]


class nulpa_opts(C.Structure):
    _fields_ = [("tolerance", C.c_double), ("max_iterations", C.c_int32),
                ("pl_period", C.c_int32), ("cc_period", C.c_int32), ("strategy", C.c_int32),
                ("switch_degree", C.c_uint32), ("precision", C.c_int32), ("exec", C.c_int32),
                ("workers", C.c_int32), ("seed", C.c_uint64), ("prune", C.c_int32),
                ("device", C.c_int32)]


class nulpa_tuning(C.Structure):
    _fields_ = [("thread_max_degree", C.c_uint32), ("warp_max_degree", C.c_uint32),
                ("block_max_degree", C.c_uint32), ("hub_chunk", C.c_uint32),
                ("async_first_pass", C.c_uint32), ("profile", C.c_uint32),
                ("schedule", C.c_uint32), ("no_identity_first", C.c_uint32),
                ("unbatched", C.c_uint32)]

NULPA_TIERS = 10
TIER_NAMES = ["thread", "half_warp", "warp", "team32", "team128", "team256", "cta512",
              "wide", "hub", "other"]


class nulpa_stats(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32),
                ("pl_iterations", C.c_int32), ("reserved", C.c_int32),
                ("cc_reverts", C.c_uint64), ("elapsed_seconds", C.c_double),
                ("delta_n", C.POINTER(C.c_uint64)), ("processed_vertices", C.c_uint64),
                ("processed_edges", C.c_uint64), ("wake_edges", C.c_uint64),
                ("algorithmic_bytes", C.c_uint64), ("setup_seconds", C.c_double),
                ("kernel_launches", C.c_uint64), ("tier_ms", C.c_double * 10),
                ("tier_bytes", C.c_double * 10), ("tier_edges", C.c_uint64 * 10),
                ("tier_passes", C.c_uint32 * 10), ("reserved2", C.c_uint32)]


class nulpa_edge_list(C.Structure):
    _fields_ = [("ne", C.c_uint64), ("n_declared", C.c_int64), ("u", C.POINTER(C.c_uint32)),
                ("v", C.POINTER(C.c_uint32)), ("w", C.POINTER(C.c_double))]


class nulpa_pass_info(C.Structure):
    _fields_ = [("changed", C.c_uint64), ("processed_vertices", C.c_uint64),
                ("processed_edges", C.c_uint64), ("wake_edges", C.c_uint64),
                ("device_ms", C.c_double), ("kernel_launches", C.c_uint64)]


class NulpaError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


_lib: C.CDLL | None = None

_SIGS = {
    "nulpa_last_error": (C.c_char_p, []),
    "nulpa_version": (C.c_int, []),
    "nulpa_default_opts": (None, [C.POINTER(nulpa_opts)]),
    "nulpa_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "nulpa_run": (C.c_int, [C.POINTER(nulpa_csr), C.POINTER(nulpa_opts), C.POINTER(nulpa_tuning),
                            C.c_void_p, C.POINTER(nulpa_stats)]),
    "nulpa_sync_step": (C.c_int, [C.POINTER(nulpa_csr), C.c_void_p, C.c_int, C.c_int, C.c_int,
                                  C.c_void_p, C.POINTER(C.c_uint64)]),
    "nulpa_modularity": (C.c_int, [C.POINTER(nulpa_csr), C.c_void_p, C.POINTER(C.c_double)]),
    "nulpa_community_count": (C.c_int, [C.POINTER(nulpa_csr), C.c_void_p,
                                        C.POINTER(C.c_uint64)]),
    "nulpa_cross_check": (C.c_int, [C.POINTER(nulpa_csr), C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.POINTER(C.c_uint64)]),
    "nulpa_partition_by_degree": (C.c_int, [C.POINTER(nulpa_csr), C.c_uint32, C.c_void_p,
                                            C.POINTER(C.c_uint64), C.c_void_p,
                                            C.POINTER(C.c_uint64)]),
    "nulpa_graph_upload": (C.c_int, [C.POINTER(nulpa_csr), C.c_int, C.POINTER(C.c_void_p)]),
    "nulpa_graph_wrap_device": (C.c_int, [C.POINTER(nulpa_csr), C.c_int, C.POINTER(C.c_void_p)]),
    "nulpa_graph_free": (C.c_int, [C.c_void_p]),
    "nulpa_graph_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint32), C.POINTER(C.c_uint64),
                                   C.POINTER(C.c_uint32), C.POINTER(C.c_int)]),
    "nulpa_graph_device_csr": (C.c_int, [C.c_void_p, C.POINTER(nulpa_csr)]),
    "nulpa_set_default_layout": (C.c_int, [C.c_int]),
    "nulpa_graph_layout": (C.c_int, [C.c_void_p, C.POINTER(C.c_int)]),
    "nulpa_graph_labels_to_vertex_order": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "nulpa_graph_labels_to_position_order": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "nulpa_graph_download": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "nulpa_run_graph": (C.c_int, [C.c_void_p, C.POINTER(nulpa_opts), C.POINTER(nulpa_tuning),
                                  C.c_void_p, C.c_void_p, C.POINTER(nulpa_stats)]),
    "nulpa_sync_step_graph": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                        C.c_void_p, C.POINTER(C.c_uint64)]),
    "nulpa_modularity_graph": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_double)]),
    "nulpa_community_count_graph": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64)]),
    "nulpa_gen_rmat": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint64, C.c_int,
                                 C.POINTER(C.c_void_p)]),
    "nulpa_gen_grid": (C.c_int, [C.c_uint32, C.c_uint32, C.c_int, C.POINTER(C.c_void_p)]),
    "nulpa_gen_web": (C.c_int, [C.c_uint32, C.c_uint64, C.c_double, C.c_uint32, C.c_uint32,
                                C.c_uint64, C.c_int, C.POINTER(C.c_void_p)]),
    "nulpa_graph_from_edges": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_int,
                                         C.POINTER(C.c_void_p)]),
    "nulpa_graph_edge_ranges": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p]),
    "nulpa_community_stats": (C.c_int, [C.POINTER(nulpa_csr), C.c_void_p, C.POINTER(C.c_uint64),
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.POINTER(C.c_uint64)]),
    "nulpa_community_stats_graph": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64),
                                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                              C.c_void_p, C.POINTER(C.c_uint64)]),
    "nulpa_load_edge_list": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(nulpa_edge_list)]),
    "nulpa_edge_list_free": (None, [C.POINTER(nulpa_edge_list)]),
    "nulpa_graph_from_edge_list": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64,
                                             C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "nulpa_graph_load": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "nulpa_session_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "nulpa_session_pack_changes": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p]),
    "nulpa_session_apply_changes": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]),
    "nulpa_graph_slice": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(C.c_void_p)]),
    "nulpa_graph_download_raw": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "nulpa_graph_download_layout": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p,
                                              C.POINTER(C.c_int)]),
    "nulpa_graph_upload_positioned": (C.c_int, [C.POINTER(nulpa_csr), C.c_void_p, C.c_void_p,
                                                C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "nulpa_community_sums_graph": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "nulpa_write_edge_list": (C.c_int, [C.c_char_p, C.POINTER(nulpa_csr)]),
    "nulpa_write_membership": (C.c_int, [C.c_char_p, C.c_void_p, C.c_uint64, C.c_int]),
    "nulpa_read_membership": (C.c_int, [C.c_char_p, C.c_uint32, C.c_void_p]),
    "nulpa_session_create": (C.c_int, [C.c_void_p, C.POINTER(nulpa_opts),
                                       C.POINTER(nulpa_tuning), C.c_uint32, C.c_uint32,
                                       C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
    "nulpa_session_init": (C.c_int, [C.c_void_p]),
    "nulpa_session_pass": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.POINTER(nulpa_pass_info)]),
    "nulpa_session_free": (C.c_int, [C.c_void_p]),
}


def exported_symbols() -> list[str]:
    return sorted(_SIGS)


def lib() -> C.CDLL:
    """Load libnulpa.so (once). Raises if it has not been built."""
    global _lib
    if _lib is None:
        path = Path(os.environ.get("NULPA_LIB", LIB_PATH))
        if not path.exists():
            raise ImportError(f"{path} is missing: build it with "
                              "`python -m paper_2411_11468_b200.build` (no CPU fallback exists)")
        L = C.CDLL(str(path))
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != NULPA_OK:
        msg = lib().nulpa_last_error().decode(errors="replace")
        from . import labelprop as lp  # error taxonomy lives with the host mirror
        if rc == NULPA_EINVAL:
            raise lp.ValidationError(msg)
        if rc == NULPA_ENOMEM:
            raise MemoryError(msg)
        if rc == NULPA_EINTERNAL:
            raise lp.InternalError(msg)
        if rc == NULPA_EFORMAT:
            raise lp.FormatError(msg)
        raise NulpaError(rc, msg)
