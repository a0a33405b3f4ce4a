"""TEST INFRASTRUCTURE ONLY — the checkers for the CUDA product.

Two independent CPU checkers of the reference ν-LPA hot path:

* ``port``: our C restatement (oracle/oracle.c -> oracle/liboracle.so), each function
  citing the reference file:line it follows;
* ``ref``: the UNMODIFIED reference library (/root/reference/proj/src/*.cpp) compiled
  by oracle/Makefile into oracle/_ref/libnulpa_ref.so, exposed through the array-only
  shim oracle/ref_shim.cpp.

Only tests/, __graft_entry__.smoke() (as the checker) and bench.py's cpu_baseline /
``--impl reference`` leg may import this package. The product (paper_2411_11468_b200)
never does.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_LIB = HERE / "liboracle.so"
REF_LIB = HERE / "_ref" / "libnulpa_ref.so"


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _p(a):
    return a.ctypes.data if a is not None and a.size else None


# --------------------------------------------------------------------------------------
# C restatement (port)


class _OrCsr(C.Structure):
    _fields_ = [("n", C.c_uint32), ("m2", C.c_uint64), ("offsets", C.c_void_p),
                ("targets", C.c_void_p), ("weights", C.c_void_p)]


class _OrConfig(C.Structure):
    _fields_ = [("tolerance", C.c_double), ("max_iterations", C.c_int32),
                ("pl_period", C.c_int32), ("cc_period", C.c_int32), ("strategy", C.c_int32),
                ("switch_degree", C.c_uint32), ("precision_bits", C.c_int32),
                ("exec", C.c_int32), ("prune", C.c_int32)]


class _OrStats(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32),
                ("pl_iterations", C.c_int32), ("pad", C.c_int32), ("cc_reverts", C.c_uint64),
                ("delta_n", C.c_uint64 * 256)]


_port = None


def port() -> C.CDLL:
    global _port
    if _port is None:
        if not PORT_LIB.exists():
            subprocess.run(["make", "-s", "-C", str(HERE), "oracle"], check=True)
        L = C.CDLL(str(PORT_LIB))
        L.or_sync_step.restype = C.c_uint64
        L.or_sync_step.argtypes = [C.POINTER(_OrCsr), C.c_void_p, C.c_int, C.c_int, C.c_int,
                                   C.c_void_p]
        L.or_lpa.restype = C.c_int
        L.or_lpa.argtypes = [C.POINTER(_OrCsr), C.POINTER(_OrConfig), C.c_void_p,
                             C.POINTER(_OrStats)]
        L.or_modularity.restype = C.c_double
        L.or_modularity.argtypes = [C.POINTER(_OrCsr), C.c_void_p]
        L.or_cross_check.restype = C.c_uint64
        L.or_cross_check.argtypes = [C.POINTER(_OrCsr), C.c_void_p, C.c_void_p, C.c_void_p]
        L.or_partition_by_degree.restype = C.c_uint64
        L.or_partition_by_degree.argtypes = [C.POINTER(_OrCsr), C.c_uint32, C.c_void_p,
                                             C.c_void_p]
        L.or_geometry.restype = C.c_int
        L.or_geometry.argtypes = [C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.or_ht_accumulate_seq.restype = C.c_uint64
        L.or_ht_accumulate_seq.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_void_p,
                                           C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]
        _port = L
    return _port


class PortGraph:
    """Keeps the numpy arrays alive for an or_csr view."""

    def __init__(self, offsets, targets, weights=None):
        self.offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        self.targets = np.ascontiguousarray(targets, dtype=np.uint32)
        self.weights = None if weights is None else np.ascontiguousarray(weights, np.float32)
        self.c = _OrCsr(self.offsets.size - 1, self.targets.size, self.offsets.ctypes.data,
                        _p(self.targets), _p(self.weights))

    @property
    def n(self):
        return int(self.offsets.size - 1)


def port_sync_step(g: PortGraph, labels, pick_less, strategy=3, precision=32):
    lin = _u32(labels)
    out = np.empty_like(lin)
    changed = port().or_sync_step(C.byref(g.c), _p(lin), int(pick_less), strategy, precision,
                                  _p(out))
    return out, int(changed)


def port_lpa(g: PortGraph, *, exec_mode=2, tolerance=0.05, max_iterations=20, pl_period=4,
             cc_period=0, strategy=3, switch_degree=32, precision=32, prune=True):
    cfg = _OrConfig(tolerance, max_iterations, pl_period, cc_period, strategy, switch_degree,
                    precision, exec_mode, 1 if prune else 0)
    labels = np.empty(g.n, dtype=np.uint32)
    st = _OrStats()
    rc = port().or_lpa(C.byref(g.c), C.byref(cfg), _p(labels), C.byref(st))
    if rc != 0:
        raise ValueError(f"or_lpa rc={rc}")
    return labels, {"iterations": st.iterations, "converged": bool(st.converged),
                    "pl_iterations": st.pl_iterations, "cc_reverts": int(st.cc_reverts),
                    "delta_n": [int(x) for x in st.delta_n[:min(st.iterations, 256)]]}


def port_modularity(g: PortGraph, labels) -> float:
    return float(port().or_modularity(C.byref(g.c), _p(_u32(labels))))


def port_cross_check(g: PortGraph, labels: np.ndarray, prev, flags: np.ndarray) -> int:
    return int(port().or_cross_check(C.byref(g.c), _p(labels), _p(_u32(prev)), _p(flags)))


def port_partition(g: PortGraph, switch_degree: int):
    low = np.empty(g.n, np.uint32)
    high = np.empty(g.n, np.uint32)
    nl = int(port().or_partition_by_degree(C.byref(g.c), switch_degree, _p(low), _p(high)))
    return low[:nl].copy(), high[:g.n - nl].copy()


def port_geometry(degree: int):
    p1, p2 = C.c_uint64(), C.c_uint64()
    rc = port().or_geometry(degree, C.byref(p1), C.byref(p2))
    return None if rc else (p1.value, p2.value)


def port_ht_seq(p1, p2, strategy, keys, values):
    k = _u32(keys)
    v = np.ascontiguousarray(values, dtype=np.float32)
    sk = np.empty(p1, np.uint32)
    sv = np.empty(p1, np.float32)
    f = port().or_ht_accumulate_seq(p1, p2, strategy, _p(k), _p(v), k.size, _p(sk), _p(sv))
    return sk, sv, int(f)


# --------------------------------------------------------------------------------------
# The reference library itself (oracle/_ref)


class _RefStats(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32),
                ("pl_iterations", C.c_int32), ("pad", C.c_int32), ("cc_reverts", C.c_uint64),
                ("elapsed_seconds", C.c_double)]


_ref = None


def ref_available() -> bool:
    return REF_LIB.exists()


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not REF_LIB.exists():
            raise FileNotFoundError(f"{REF_LIB} not built (needs /root/reference at build time)")
        L = C.CDLL(str(REF_LIB))
        vp = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        for name, res, args in [
            ("ref_graph_from_csr", vp, [vp, vp, vp, C.c_uint32, C.c_uint64]),
            ("ref_graph_from_edges", vp, [vp, vp, vp, C.c_uint64, C.c_int64, C.c_int]),
            ("ref_load_graph", C.c_int64, [C.c_char_p, C.c_int, C.c_uint64, vp, vp, vp,
                                           C.POINTER(C.c_int64)]),
            ("ref_graph_planted", vp, [C.c_uint32, C.c_uint32, C.c_double, C.c_double,
                                       C.c_uint64, vp]),
            ("ref_planted_edges", C.c_int64, [C.c_uint32, C.c_uint32, C.c_double, C.c_double,
                                              C.c_uint64, vp, vp, C.c_uint64]),
            ("ref_graph_star", vp, [C.c_uint32]),
            ("ref_graph_ring_of_cliques", vp, [C.c_uint32, C.c_uint32]),
            ("ref_graph_free", None, [vp]),
            ("ref_graph_order", C.c_uint32, [vp]),
            ("ref_graph_m2", C.c_uint64, [vp]),
            ("ref_graph_total_2m", C.c_double, [vp]),
            ("ref_graph_arrays", None, [vp, vp, vp, vp]),
            ("ref_lpa", C.c_int, [vp, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint32,
                                  C.c_int, C.c_int, C.c_int, C.c_int, vp, vp,
                                  C.POINTER(_RefStats)]),
            ("ref_sync_step", C.c_int, [vp, vp, C.c_int, C.c_int, C.c_int, vp,
                                        C.POINTER(C.c_uint64)]),
            ("ref_modularity", C.c_int, [vp, vp, C.POINTER(C.c_double)]),
            ("ref_community_count", C.c_int, [vp, vp, C.POINTER(C.c_uint64)]),
            ("ref_cross_check", C.c_int, [vp, vp, vp, vp, C.POINTER(C.c_uint64)]),
            ("ref_lpa_move", C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_uint32,
                                       C.POINTER(C.c_uint64)]),
            ("ref_partition_by_degree", C.c_int, [vp, C.c_uint32, vp, C.POINTER(C.c_uint64), vp,
                                                  C.POINTER(C.c_uint64)]),
            ("ref_geometry", C.c_int, [vp, C.c_uint32, C.POINTER(C.c_uint64),
                                       C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
            ("ref_ht_accumulate_seq", C.c_uint64, [C.c_uint64, C.c_uint64, C.c_int, vp, vp,
                                                   C.c_uint64, vp, vp]),
            ("ref_reference_lpa", C.c_int, [vp, C.c_double, C.c_int, C.c_int, vp, vp,
                                            C.POINTER(C.c_int), C.POINTER(C.c_int)]),
            ("ref_modularity_oracle", C.c_int, [vp, vp, C.POINTER(C.c_double)]),
            ("ref_hardware_concurrency", C.c_uint32, []),
            ("ref_write_edge_list", C.c_int, [vp, C.c_char_p]),
            ("ref_write_membership", C.c_int, [C.c_char_p, vp, C.c_uint64]),
            ("ref_read_membership", C.c_int, [C.c_char_p, C.c_uint32, vp]),
        ]:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _ref = L
    return _ref


class RefGraph:
    """A labelprop_ref::CsrGraph owned by the reference library."""

    def __init__(self, handle):
        if not handle:
            raise ValueError(ref().ref_last_error().decode())
        self.h = C.c_void_p(handle)
        self.n = int(ref().ref_graph_order(self.h))
        self.m2 = int(ref().ref_graph_m2(self.h))

    @classmethod
    def from_csr(cls, offsets, targets, weights=None):
        o = np.ascontiguousarray(offsets, np.uint64)
        t = _u32(targets)
        w = None if weights is None else np.ascontiguousarray(weights, np.float32)
        return cls(ref().ref_graph_from_csr(_p(o), _p(t), _p(w), o.size - 1, t.size))

    @classmethod
    def from_edges(cls, u, v, w=None, n_declared=-1, symmetrize=True):
        u, v = _u32(u), _u32(v)
        wd = None if w is None else np.ascontiguousarray(w, np.float64)
        return cls(ref().ref_graph_from_edges(_p(u), _p(v), _p(wd), u.size, n_declared,
                                              int(symmetrize)))

    @classmethod
    def planted(cls, n, communities, p_in, p_out, seed):
        gt = np.empty(n, np.uint32)
        g = cls(ref().ref_graph_planted(n, communities, p_in, p_out, seed, _p(gt)))
        g.ground_truth = gt
        return g

    @classmethod
    def star(cls, leaves):
        return cls(ref().ref_graph_star(leaves))

    @classmethod
    def ring_of_cliques(cls, cliques, size):
        return cls(ref().ref_graph_ring_of_cliques(cliques, size))

    def arrays(self):
        o = np.empty(self.n + 1, np.uint64)
        t = np.empty(self.m2, np.uint32)
        w = np.empty(self.m2, np.float32)
        ref().ref_graph_arrays(self.h, _p(o), _p(t), _p(w))
        return o, t, w

    def __del__(self):
        try:
            ref().ref_graph_free(self.h)
        except Exception:
            pass


def _ref_check(rc):
    if rc != 0:
        raise ValueError(f"reference rc={rc}: {ref().ref_last_error().decode()}")


def ref_lpa(g: RefGraph, *, exec_mode=0, tolerance=0.05, max_iterations=20, pl_period=4,
            cc_period=0, strategy=3, switch_degree=32, precision=32, workers=0, prune=True):
    labels = np.empty(g.n, np.uint32)
    dn = np.zeros(max(1, max_iterations), np.uint64)
    st = _RefStats()
    _ref_check(ref().ref_lpa(g.h, tolerance, max_iterations, pl_period, cc_period, strategy,
                             switch_degree, precision, exec_mode, workers, int(prune),
                             _p(labels), _p(dn), C.byref(st)))
    return labels, {"iterations": st.iterations, "converged": bool(st.converged),
                    "pl_iterations": st.pl_iterations, "cc_reverts": int(st.cc_reverts),
                    "elapsed_seconds": st.elapsed_seconds,
                    "delta_n": [int(x) for x in dn[:st.iterations]]}


def ref_sync_step(g: RefGraph, labels, pick_less, strategy=3, precision=32):
    lin = _u32(labels)
    out = np.empty_like(lin)
    ch = C.c_uint64()
    _ref_check(ref().ref_sync_step(g.h, _p(lin), int(pick_less), strategy, precision, _p(out),
                                   C.byref(ch)))
    return out, int(ch.value)


def ref_modularity(g: RefGraph, labels) -> float:
    q = C.c_double()
    _ref_check(ref().ref_modularity(g.h, _p(_u32(labels)), C.byref(q)))
    return q.value


def ref_community_count(g: RefGraph, labels) -> int:
    c = C.c_uint64()
    _ref_check(ref().ref_community_count(g.h, _p(_u32(labels)), C.byref(c)))
    return int(c.value)


def ref_cross_check(g: RefGraph, labels: np.ndarray, prev, flags: np.ndarray) -> int:
    r = C.c_uint64()
    _ref_check(ref().ref_cross_check(g.h, _p(labels), _p(_u32(prev)), _p(flags), C.byref(r)))
    return int(r.value)


def ref_partition(g: RefGraph, switch_degree):
    low = np.empty(g.n, np.uint32)
    high = np.empty(g.n, np.uint32)
    nl, nh = C.c_uint64(), C.c_uint64()
    _ref_check(ref().ref_partition_by_degree(g.h, switch_degree, _p(low), C.byref(nl), _p(high),
                                             C.byref(nh)))
    return low[:nl.value].copy(), high[:nh.value].copy()


def ref_ht_seq(p1, p2, strategy, keys, values):
    k = _u32(keys)
    v = np.ascontiguousarray(values, np.float32)
    sk = np.empty(p1, np.uint32)
    sv = np.empty(p1, np.float32)
    f = ref().ref_ht_accumulate_seq(p1, p2, strategy, _p(k), _p(v), k.size, _p(sk), _p(sv))
    return sk, sv, int(f)


def ref_modularity_oracle(g: RefGraph, labels) -> float:
    q = C.c_double()
    _ref_check(ref().ref_modularity_oracle(g.h, _p(_u32(labels)), C.byref(q)))
    return q.value


def ref_load_graph(path, fmt):
    """labelprop_ref::load_graph -> (u, v, w, n_declared) in listing order, or raises
    ValueError('F:<message>') / ValueError('V:<message>')."""
    nd = C.c_int64()
    ne = ref().ref_load_graph(str(path).encode(), fmt, 0, None, None, None, C.byref(nd))
    if ne < 0:
        raise ValueError(ref().ref_last_error().decode())
    u = np.empty(ne, np.uint32)
    v = np.empty(ne, np.uint32)
    w = np.empty(ne, np.float64)
    ref().ref_load_graph(str(path).encode(), fmt, ne, _p(u), _p(v), _p(w), C.byref(nd))
    return u, v, w, nd.value


# The reference's ofstream writers crash once numpy's bundled runtime libraries are in the
# process (a libstdc++/libgfortran interaction, reproducible with ctypes alone), so they
# run in a child interpreter that loads only ctypes.
_WRITER = r"""
import ctypes as C, sys
L = C.CDLL(sys.argv[1])
def load(path, ct):
    raw = open(path, "rb").read()
    return (ct * (len(raw) // C.sizeof(ct))).from_buffer_copy(raw)
L.ref_last_error.restype = C.c_char_p
if sys.argv[2] == "edges":
    o, t, w = load(sys.argv[3], C.c_uint64), load(sys.argv[4], C.c_uint32), load(sys.argv[5], C.c_float)
    L.ref_graph_from_csr.restype = C.c_void_p
    g = C.c_void_p(L.ref_graph_from_csr(o, t, w, C.c_uint32(len(o) - 1), C.c_uint64(len(t))))
    rc = L.ref_write_edge_list(g, sys.argv[6].encode())
else:
    lab = load(sys.argv[3], C.c_uint32)
    rc = L.ref_write_membership(sys.argv[4].encode(), lab, C.c_uint64(len(lab)))
if rc:
    sys.stderr.write(L.ref_last_error().decode()); sys.exit(3)
"""


def _run_writer(*args):
    import subprocess
    import sys
    r = subprocess.run([sys.executable, "-c", _WRITER, str(REF_LIB), *map(str, args)],
                       capture_output=True, text=True)
    if r.returncode:
        raise ValueError(r.stderr.strip() or f"reference writer failed ({r.returncode})")


def ref_write_edge_list(g: "RefGraph", path):
    """labelprop_ref::write_edge_list (graph.cpp:309-325)."""
    import tempfile
    o, t, w = g.arrays()
    with tempfile.TemporaryDirectory() as d:
        files = [f"{d}/{k}.bin" for k in "otw"]
        for f, a in zip(files, (o, t, w)):
            a.tofile(f)
        _run_writer("edges", *files, path)


def ref_write_membership(path, labels):
    """labelprop_ref::write_membership (io.cpp:9-14)."""
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        _u32(labels).tofile(f"{d}/l.bin")
        _run_writer("membership", f"{d}/l.bin", path)


def ref_read_membership(path, n):
    """labelprop_ref::read_membership (io.cpp:16-56), or ValueError('F:..'/'V:..')."""
    out = np.zeros(n, np.uint32)
    if ref().ref_read_membership(str(path).encode(), n, _p(out)) != 0:
        raise ValueError(ref().ref_last_error().decode())
    return out


def ref_planted_edges(n, communities, p_in, p_out, seed):
    ne = int(ref().ref_planted_edges(n, communities, p_in, p_out, seed, None, None, 0))
    u = np.empty(ne, np.uint32)
    v = np.empty(ne, np.uint32)
    ref().ref_planted_edges(n, communities, p_in, p_out, seed, _p(u), _p(v), ne)
    return u, v
