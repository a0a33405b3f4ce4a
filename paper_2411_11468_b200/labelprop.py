"""Host-side mirror of the reference's ``labelprop`` engine API over the nulpa C ABI.

Same names, argument meaning and error behaviour as the reference C++
(paths relative to /root/reference/proj):

    CsrGraph             include/labelprop/graph.hpp:53-84 (ctor check graph.cpp:165-172)
    LpaConfig / RunStats / LpaResult   include/labelprop/lpa.hpp:25-51
    ExecMode / ValuePrecision / ProbeStrategy   lpa.hpp:20-23, hashtable.hpp:25
    lpa                  lpa.hpp:84           -> nulpa_run
    partition_by_degree  lpa.hpp:63           -> nulpa_partition_by_degree
    cross_check          lpa.hpp:72-73        -> nulpa_cross_check
    modularity           quality.hpp:19       -> nulpa_modularity
    ValidationError / InternalError           graph.hpp:17-31

Every compute call runs CUDA kernels; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

from . import _capi


class FormatError(ValueError):
    """labelprop::FormatError (graph.hpp:17-19): a malformed input file."""


class ValidationError(ValueError):
    """labelprop::ValidationError (graph.hpp:23-25)."""


class InternalError(RuntimeError):
    """labelprop::InternalError (graph.hpp:29-31)."""


class ExecMode(IntEnum):
    ParallelAsync = 0
    Sequential = 1
    Synchronous = 2


class ValuePrecision(IntEnum):
    Bits32 = 32
    Bits64 = 64


class ProbeStrategy(IntEnum):
    Linear = 0
    Quadratic = 1
    DoubleHash = 2
    QuadraticDouble = 3


@dataclass
class LpaConfig:
    tolerance: float = 0.05
    max_iterations: int = 20
    pl_period: int = 4
    cc_period: int = 0
    strategy: ProbeStrategy = ProbeStrategy.QuadraticDouble
    switch_degree: int = 32
    precision: ValuePrecision = ValuePrecision.Bits32
    exec: ExecMode = ExecMode.ParallelAsync
    workers: int = 0
    seed: int = 0
    prune: bool = True


@dataclass
class RunStats:
    iterations: int = 0
    delta_n_per_iter: list[int] = field(default_factory=list)
    converged: bool = False
    pl_iterations: int = 0
    cc_reverts: int = 0
    elapsed_seconds: float = 0.0
    # device counters (not in the reference RunStats)
    processed_vertices: int = 0
    processed_edges: int = 0
    wake_edges: int = 0
    algorithmic_bytes: int = 0
    setup_seconds: float = 0.0


@dataclass
class LpaResult:
    labels: np.ndarray
    stats: RunStats


class FileFormat(IntEnum):
    """labelprop::FileFormat (graph.hpp:86)."""
    MatrixMarket = 0
    EdgeListText = 1


@dataclass
class EdgeList:
    """labelprop::EdgeList (graph.hpp:40-43) as arrays in listing order."""
    u: np.ndarray
    v: np.ndarray
    w: np.ndarray
    n_declared: int | None = None


@dataclass
class DegreePartition:
    low: np.ndarray
    high: np.ndarray


@dataclass
class Tuning:
    """Kernel-tier bounds (nulpa_tuning); 0 = library default."""
    thread_max_degree: int = 0
    warp_max_degree: int = 0
    block_max_degree: int = 0
    schedule: int = 0  # 0 default (= 4); 1 position order; 2/3 scrambled; 4 chunk walk (nulpa.h)
    profile: bool = False
    identity_first: bool = True  # table-free first pass from identity labels
    async_first_pass: int = 0  # 1: ParallelAsync pass 0 as the table-free synchronous pass
    batched: bool = True  # passes enqueued in batches behind the device convergence guard

    def to_c(self) -> _capi.nulpa_tuning:
        t = _capi.nulpa_tuning()
        t.thread_max_degree = self.thread_max_degree
        t.warp_max_degree = self.warp_max_degree
        t.block_max_degree = self.block_max_degree
        t.schedule = self.schedule
        t.profile = 1 if self.profile else 0
        t.no_identity_first = 0 if self.identity_first else 1
        t.async_first_pass = self.async_first_pass
        t.unbatched = 0 if self.batched else 1
        return t


class CsrGraph:
    """Host CSR (offsets u64[n+1], targets u32[m2], weights f32[m2])."""

    def __init__(self, offsets, targets, weights=None):
        self.offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        self.targets = np.ascontiguousarray(targets, dtype=np.uint32)
        if weights is None:
            weights = np.ones(self.targets.shape[0], dtype=np.float32)
        self.weights = np.ascontiguousarray(weights, dtype=np.float32)
        if (self.offsets.size == 0 or int(self.offsets[-1]) != self.targets.size
                or self.targets.size != self.weights.size):
            raise ValidationError("inconsistent CSR arrays")
        self._total_2m = float(self.weights.astype(np.float64).sum())

    def order(self) -> int:
        return int(self.offsets.size - 1)

    def directed_size(self) -> int:
        return int(self.targets.size)

    def degree(self, i: int) -> int:
        return int(self.offsets[i + 1] - self.offsets[i])

    def total_weight_2m(self) -> float:
        return self._total_2m

    def neighbors(self, i: int) -> np.ndarray:
        return self.targets[self.offsets[i]:self.offsets[i + 1]]

    def csr_view(self) -> _capi.nulpa_csr:
        c = _capi.nulpa_csr()
        c.n = self.order()
        c.m2 = self.directed_size()
        c.offsets = self.offsets.ctypes.data
        c.targets = self.targets.ctypes.data if self.targets.size else None
        c.weights = self.weights.ctypes.data if self.weights.size else None
        return c


def _opts(cfg: LpaConfig, device: int = 0) -> _capi.nulpa_opts:
    o = _capi.nulpa_opts()
    _capi.lib().nulpa_default_opts(C.byref(o))
    o.tolerance = cfg.tolerance
    o.max_iterations = int(cfg.max_iterations)
    o.pl_period = int(cfg.pl_period)
    o.cc_period = int(cfg.cc_period)
    o.strategy = int(cfg.strategy)
    o.switch_degree = int(cfg.switch_degree) & 0xFFFFFFFF
    o.precision = int(cfg.precision)
    o.exec = int(cfg.exec)
    o.workers = int(cfg.workers)
    o.seed = int(cfg.seed)
    o.prune = 1 if cfg.prune else 0
    o.device = device
    return o


def _stats(st: _capi.nulpa_stats, dn: np.ndarray) -> RunStats:
    return RunStats(iterations=st.iterations,
                    delta_n_per_iter=[int(x) for x in dn[:st.iterations]],
                    converged=bool(st.converged), pl_iterations=st.pl_iterations,
                    cc_reverts=int(st.cc_reverts), elapsed_seconds=st.elapsed_seconds,
                    processed_vertices=int(st.processed_vertices),
                    processed_edges=int(st.processed_edges), wake_edges=int(st.wake_edges),
                    algorithmic_bytes=int(st.algorithmic_bytes),
                    setup_seconds=st.setup_seconds)


def _ptr(a: np.ndarray):
    return a.ctypes.data if a.size else None


def lpa(g: CsrGraph, config: LpaConfig | None = None, tuning: Tuning | None = None,
        device: int = 0) -> LpaResult:
    """labelprop::lpa (lpa.hpp:84): host buffers in, host labels out."""
    cfg = config or LpaConfig()
    o = _opts(cfg, device)
    labels = np.empty(g.order(), dtype=np.uint32)
    dn = np.zeros(max(1, int(cfg.max_iterations)), dtype=np.uint64)
    st = _capi.nulpa_stats()
    st.delta_n = dn.ctypes.data_as(C.POINTER(C.c_uint64))
    csr = g.csr_view()
    t = tuning.to_c() if tuning else None
    _capi.check(_capi.lib().nulpa_run(C.byref(csr), C.byref(o), C.byref(t) if t else None,
                                      _ptr(labels), C.byref(st)))
    return LpaResult(labels=labels, stats=_stats(st, dn))


def sync_step(g: CsrGraph, labels_in, pick_less: bool, strategy: int = 3,
              precision: int = 32) -> tuple[np.ndarray, int]:
    """One synchronous label-choice step over every vertex of degree >= 1."""
    lin = np.ascontiguousarray(labels_in, dtype=np.uint32)
    out = np.empty_like(lin)
    changed = C.c_uint64()
    csr = g.csr_view()
    _capi.check(_capi.lib().nulpa_sync_step(C.byref(csr), _ptr(lin), int(pick_less),
                                            int(strategy), int(precision), _ptr(out),
                                            C.byref(changed)))
    return out, int(changed.value)


def modularity(g: CsrGraph, labels) -> float:
    """labelprop::modularity (quality.hpp:19)."""
    lab = np.ascontiguousarray(labels, dtype=np.uint32)
    if lab.size != g.order():
        raise ValidationError(f"labeling has {lab.size} entries for {g.order()} vertices")
    q = C.c_double()
    csr = g.csr_view()
    _capi.check(_capi.lib().nulpa_modularity(C.byref(csr), _ptr(lab), C.byref(q)))
    return q.value


def community_count(g: CsrGraph, labels) -> int:
    """labelprop::community_stats(...).count (quality.cpp:56-78)."""
    lab = np.ascontiguousarray(labels, dtype=np.uint32)
    cnt = C.c_uint64()
    csr = g.csr_view()
    _capi.check(_capi.lib().nulpa_community_count(C.byref(csr), _ptr(lab), C.byref(cnt)))
    return int(cnt.value)


def load_graph(path, fmt: FileFormat) -> EdgeList:
    """labelprop::load_graph (graph.hpp:95-96): FormatError / ValidationError as the reference."""
    el = _capi.nulpa_edge_list()
    _capi.check(_capi.lib().nulpa_load_edge_list(str(path).encode(), int(fmt), C.byref(el)))
    try:
        ne = int(el.ne)
        u = np.ctypeslib.as_array(el.u, (ne,)).copy() if ne else np.empty(0, np.uint32)
        v = np.ctypeslib.as_array(el.v, (ne,)).copy() if ne else np.empty(0, np.uint32)
        w = np.ctypeslib.as_array(el.w, (ne,)).copy() if ne else np.empty(0, np.float64)
        nd = int(el.n_declared)
    finally:
        _capi.lib().nulpa_edge_list_free(C.byref(el))
    return EdgeList(u, v, w, None if nd < 0 else nd)


def build_csr(el: EdgeList, symmetrize: bool, device: int = 0) -> CsrGraph:
    """labelprop::build_csr (graph.hpp:107), built on the device (bit-exact)."""
    dg = DeviceGraph.from_edge_list(el, symmetrize, device)
    try:
        return dg.download()
    finally:
        dg.free()


@dataclass
class CommunityStats:
    """labelprop::CommunityStats (quality.hpp:32-38)."""
    count: int
    size_histogram: dict
    sigma: dict
    big_sigma: dict


def community_stats(g: CsrGraph, labels) -> CommunityStats:
    """labelprop::community_stats (quality.cpp:56-78), on the device."""
    lab = np.ascontiguousarray(labels, dtype=np.uint32)
    if lab.size != g.order():
        raise ValidationError(f"labeling has {lab.size} entries for {g.order()} vertices")
    n = max(1, g.order())
    comm = np.empty(n, np.uint32)
    sg = np.empty(n, np.float64)
    bg = np.empty(n, np.float64)
    hs = np.empty(n, np.uint64)
    hc = np.empty(n, np.uint64)
    cnt, hl = C.c_uint64(), C.c_uint64()
    csr = g.csr_view()
    _capi.check(_capi.lib().nulpa_community_stats(C.byref(csr), _ptr(lab), C.byref(cnt),
                                                  _ptr(comm), _ptr(sg), _ptr(bg), _ptr(hs),
                                                  _ptr(hc), C.byref(hl)))
    k, h = int(cnt.value), int(hl.value)
    return CommunityStats(k, {int(a): int(b) for a, b in zip(hs[:h], hc[:h])},
                          {int(c): float(x) for c, x in zip(comm[:k], sg[:k])},
                          {int(c): float(x) for c, x in zip(comm[:k], bg[:k])})


def delta_modularity(m: float, ki: float, ki_to_c: float, ki_to_d: float, sigma_c: float,
                     sigma_d: float) -> float:
    """labelprop::delta_modularity (quality.cpp:51-54), closed form."""
    return (ki_to_c - ki_to_d) / m - ki * (ki + sigma_c - sigma_d) / (2.0 * m * m)


def write_membership(path, labels, device: int = 0) -> None:
    """labelprop::write_membership (io.cpp:9-14): `vertex<TAB>label` per line, the text
    formatted on the device (nulpa_write_membership, textout.cu)."""
    lab = np.ascontiguousarray(labels, dtype=np.uint32)
    _capi.check(_capi.lib().nulpa_write_membership(str(path).encode(), _ptr(lab), lab.size,
                                                   device))


def read_membership(path, n: int) -> np.ndarray:
    """labelprop::read_membership (io.cpp:16-56): same checks and messages
    (nulpa_read_membership, textio.cpp)."""
    labels = np.zeros(n, np.uint32)
    _capi.check(_capi.lib().nulpa_read_membership(str(path).encode(), n, _ptr(labels)))
    return labels


def write_edge_list(g: CsrGraph, path) -> None:
    """labelprop::write_edge_list (graph.hpp:112, graph.cpp:309-325)."""
    csr = g.csr_view()
    _capi.check(_capi.lib().nulpa_write_edge_list(str(path).encode(), C.byref(csr)))


def partition_by_degree(g: CsrGraph, switch_degree: int) -> DegreePartition:
    """labelprop::partition_by_degree (lpa.hpp:63)."""
    n = g.order()
    low = np.empty(n, dtype=np.uint32)
    high = np.empty(n, dtype=np.uint32)
    nl, nh = C.c_uint64(), C.c_uint64()
    csr = g.csr_view()
    _capi.check(_capi.lib().nulpa_partition_by_degree(C.byref(csr), int(switch_degree),
                                                      _ptr(low), C.byref(nl), _ptr(high),
                                                      C.byref(nh)))
    return DegreePartition(low=low[:nl.value].copy(), high=high[:nh.value].copy())


def cross_check(g: CsrGraph, labels: np.ndarray, prev, flags: np.ndarray) -> int:
    """labelprop::cross_check (lpa.hpp:72-73): labels and flags updated in place."""
    n = g.order()
    if labels.size != n or len(prev) != n or flags.size != n:
        raise ValidationError("cross-check label arrays must cover every vertex")
    if labels.dtype != np.uint32 or not labels.flags.c_contiguous:
        raise TypeError("labels must be a contiguous uint32 array (updated in place)")
    if flags.dtype != np.uint8 or not flags.flags.c_contiguous:
        raise TypeError("flags must be a contiguous uint8 array (updated in place)")
    pv = np.ascontiguousarray(prev, dtype=np.uint32)
    rev = C.c_uint64()
    csr = g.csr_view()
    _capi.check(_capi.lib().nulpa_cross_check(C.byref(csr), _ptr(labels), _ptr(pv), _ptr(flags),
                                              C.byref(rev)))
    return int(rev.value)


def set_default_layout(layout: int) -> None:
    """Layout of graphs created afterwards (nulpa_set_default_layout)."""
    _capi.check(_capi.lib().nulpa_set_default_layout(int(layout)))


class DeviceGraph:
    """A CSR resident in HBM (nulpa_graph). Build by upload or on-device generator.

    Rows are stored in position order (degree buckets, see include/nulpa/nulpa.h); every
    label array this class takes or returns is in vertex order."""

    def __init__(self, handle: int, device: int = 0):
        self._h = C.c_void_p(handle)
        self.device = device
        n, m2, md, w = C.c_uint32(), C.c_uint64(), C.c_uint32(), C.c_int()
        _capi.check(_capi.lib().nulpa_graph_info(self._h, C.byref(n), C.byref(m2), C.byref(md),
                                                 C.byref(w)))
        self.n, self.m2, self.max_degree, self.weighted = n.value, m2.value, md.value, bool(w.value)

    @classmethod
    def upload(cls, g: CsrGraph, device: int = 0) -> "DeviceGraph":
        h = C.c_void_p()
        csr = g.csr_view()
        _capi.check(_capi.lib().nulpa_graph_upload(C.byref(csr), device, C.byref(h)))
        return cls(h.value, device)

    @classmethod
    def rmat(cls, scale: int, edgefactor: int = 16, seed: int = 1, device: int = 0):
        h = C.c_void_p()
        _capi.check(_capi.lib().nulpa_gen_rmat(scale, edgefactor, seed, device, C.byref(h)))
        return cls(h.value, device)

    @classmethod
    def grid(cls, rows: int, cols: int, device: int = 0):
        h = C.c_void_p()
        _capi.check(_capi.lib().nulpa_gen_grid(rows, cols, device, C.byref(h)))
        return cls(h.value, device)

    @classmethod
    def web(cls, n: int, edges: int, gamma: float = 2.1, hubs: int = 8,
            hub_degree: int = 2_000_000, seed: int = 1, device: int = 0):
        h = C.c_void_p()
        _capi.check(_capi.lib().nulpa_gen_web(n, edges, gamma, hubs, hub_degree, seed, device,
                                              C.byref(h)))
        return cls(h.value, device)

    @classmethod
    def from_edge_list(cls, el: "EdgeList", symmetrize: bool = True, device: int = 0):
        """build_csr on the device (nulpa_graph_from_edge_list)."""
        u = np.ascontiguousarray(el.u, dtype=np.uint32)
        v = np.ascontiguousarray(el.v, dtype=np.uint32)
        w = None if el.w is None else np.ascontiguousarray(el.w, dtype=np.float64)
        nd = -1 if el.n_declared is None else int(el.n_declared)
        h = C.c_void_p()
        _capi.check(_capi.lib().nulpa_graph_from_edge_list(
            _ptr(u) if u.size else None, _ptr(v) if v.size else None,
            _ptr(w) if w is not None and w.size else None, u.size, nd, int(symmetrize), device,
            C.byref(h)))
        return cls(h.value, device)

    @classmethod
    def load(cls, path, fmt: "FileFormat", symmetrize: bool = True, device: int = 0):
        """load_graph + build_csr (nulpa_graph_load)."""
        h = C.c_void_p()
        _capi.check(_capi.lib().nulpa_graph_load(str(path).encode(), int(fmt), int(symmetrize),
                                                 device, C.byref(h)))
        return cls(h.value, device)

    @classmethod
    def from_edges(cls, u, v, n: int, device: int = 0):
        u = np.ascontiguousarray(u, dtype=np.uint32)
        v = np.ascontiguousarray(v, dtype=np.uint32)
        h = C.c_void_p()
        _capi.check(_capi.lib().nulpa_graph_from_edges(_ptr(u), _ptr(v), u.size, n, device,
                                                       C.byref(h)))
        return cls(h.value, device)

    def download(self) -> CsrGraph:
        off = np.empty(self.n + 1, dtype=np.uint64)
        tgt = np.empty(self.m2, dtype=np.uint32)
        w = np.empty(self.m2, dtype=np.float32) if self.weighted else None
        _capi.check(_capi.lib().nulpa_graph_download(self._h, _ptr(off), _ptr(tgt),
                                                     _ptr(w) if w is not None else None))
        return CsrGraph(off, tgt, w)

    @property
    def layout(self) -> int:
        """NULPA_LAYOUT_IDENTITY or NULPA_LAYOUT_DEGREE_BUCKETS (position-order rows)."""
        x = C.c_int()
        _capi.check(_capi.lib().nulpa_graph_layout(self._h, C.byref(x)))
        return x.value

    def labels_to_vertex_order(self, pos_ptr: int, out_ptr: int) -> None:
        """Device label array in position order (sessions) -> vertex order."""
        _capi.check(_capi.lib().nulpa_graph_labels_to_vertex_order(self._h, pos_ptr, out_ptr))

    def labels_to_position_order(self, vtx_ptr: int, out_ptr: int) -> None:
        _capi.check(_capi.lib().nulpa_graph_labels_to_position_order(self._h, vtx_ptr, out_ptr))

    def device_csr(self) -> _capi.nulpa_csr:
        """Device pointers of the resident arrays (position order, see `layout`)."""
        c = _capi.nulpa_csr()
        _capi.check(_capi.lib().nulpa_graph_device_csr(self._h, C.byref(c)))
        return c

    def lpa(self, config: LpaConfig | None = None, tuning: Tuning | None = None,
            labels_device_ptr: int | None = None, want_host: bool = True) -> LpaResult:
        cfg = config or LpaConfig()
        o = _opts(cfg, self.device)
        labels = np.empty(self.n, dtype=np.uint32) if want_host else np.empty(0, np.uint32)
        dn = np.zeros(max(1, int(cfg.max_iterations)), dtype=np.uint64)
        st = _capi.nulpa_stats()
        st.delta_n = dn.ctypes.data_as(C.POINTER(C.c_uint64))
        t = tuning.to_c() if tuning else None
        _capi.check(_capi.lib().nulpa_run_graph(self._h, C.byref(o), C.byref(t) if t else None,
                                                _ptr(labels) if want_host else None,
                                                labels_device_ptr, C.byref(st)))
        return LpaResult(labels=labels, stats=_stats(st, dn))

    def sync_step_device(self, labels_in_ptr: int, labels_out_ptr: int, pick_less: bool,
                         strategy: int = 3, precision: int = 32) -> int:
        changed = C.c_uint64()
        _capi.check(_capi.lib().nulpa_sync_step_graph(self._h, labels_in_ptr, int(pick_less),
                                                      strategy, precision, labels_out_ptr,
                                                      C.byref(changed)))
        return int(changed.value)

    def modularity_device(self, labels_ptr: int) -> float:
        q = C.c_double()
        _capi.check(_capi.lib().nulpa_modularity_graph(self._h, labels_ptr, C.byref(q)))
        return q.value

    def community_count_device(self, labels_ptr: int) -> int:
        c = C.c_uint64()
        _capi.check(_capi.lib().nulpa_community_count_graph(self._h, labels_ptr, C.byref(c)))
        return int(c.value)

    def free(self) -> None:
        if self._h:
            _capi.lib().nulpa_graph_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
