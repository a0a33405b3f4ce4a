"""Partitioned multi-GPU ν-LPA: one process per GPU, torch.distributed plumbing.

Layout: a 1-D edge-balanced partition of the resident position order (rank p owns
positions [b_p, b_{p+1}) with offsets[b_p] ~ p*m2/P, `nulpa_graph_edge_ranges`); labels
u32[n] and wake flags u8[n] are replicated on every rank, in position order
(`DeviceRangeEngine.vertex_labels` returns vertex order). Each pass:

1. every rank runs one pass over its own range (`nulpa_session_pass`): ParallelAsync
   in place inside the range, Synchronous into a staging buffer then applied;
   neighbour wake-ups write flags[j] = 0 for owned AND remote j;
2. label exchange: an all-gather-v of the owned ranges (P in-place broadcasts, root p);
3. wake exchange: remote entries are primed to 1 ("processed") before the pass, so a
   MIN-reduce of flags[range_p] to its owner p ORs every rank's wake-ups into it;
4. counters (changed, processed vertices/edges, wakes): one SUM all-reduce.

The run_engine schedule (lpa.cpp:246-315: Pick-Less every pl_period, flag reset on leaving
a PL pass or without pruning, ΔN/n < tolerance on a non-PL pass) is driven here on the host,
identically on every rank. Across ranks the passes are Jacobi (remote labels are one pass
stale); a Synchronous run is therefore bit-identical to the single-GPU Synchronous run.
Cross-check (cc_period > 0) and Sequential mode are not partitioned (ValidationError).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from .labelprop import ExecMode, LpaConfig, Tuning, ValidationError, _opts


@dataclass
class PartitionedStats:
    iterations: int = 0
    delta_n_per_iter: list[int] = field(default_factory=list)
    converged: bool = False
    pl_iterations: int = 0
    pass_ms: list[float] = field(default_factory=list)       # this rank's pass time
    exchange_ms: list[float] = field(default_factory=list)   # this rank's exchange time
    processed_edges: int = 0
    kernel_launches: int = 0


def edge_balanced_bounds(offsets: np.ndarray, parts: int) -> list[int]:
    """Host reference of nulpa_graph_edge_ranges (smallest v with offsets[v] >= p*m2/P)."""
    m2 = int(offsets[-1])
    n = offsets.size - 1
    b = [0]
    for p in range(1, parts):
        b.append(int(np.searchsorted(offsets, (m2 * p) // parts, side="left")))
    b.append(n)
    return [min(x, n) for x in b]


class DeviceRangeEngine:
    """One rank's pass engine: a nulpa_session over a DeviceGraph range, on torch tensors."""

    def __init__(self, dg, cfg: LpaConfig, lo: int, hi: int, tuning: Tuning | None = None):
        import torch
        self.n = dg.n
        self.lo, self.hi = lo, hi
        dev = f"cuda:{dg.device}"
        self.labels = torch.empty(dg.n, dtype=torch.int32, device=dev)
        self.flags = torch.empty(dg.n, dtype=torch.uint8, device=dev)
        o = _opts(cfg, dg.device)
        t = tuning.to_c() if tuning else None
        h = C.c_void_p()
        _capi.check(_capi.lib().nulpa_session_create(dg._h, C.byref(o), C.byref(t) if t else None,
                                                     lo, hi, self.labels.data_ptr(),
                                                     self.flags.data_ptr(), C.byref(h)))
        self._h = h
        self._dg = dg  # keep the graph alive

    def init(self):
        _capi.check(_capi.lib().nulpa_session_init(self._h))

    def vertex_labels(self):
        """The replicated labels (position order inside the session) in vertex order."""
        import torch
        out = torch.empty_like(self.labels)
        self._dg.labels_to_vertex_order(self.labels.data_ptr(), out.data_ptr())
        return out

    def pass_(self, pick_less: bool, wake: bool = True) -> dict:
        info = _capi.nulpa_pass_info()
        _capi.check(_capi.lib().nulpa_session_pass(self._h, int(pick_less), int(wake),
                                                   C.byref(info)))
        return {"changed": info.changed, "processed_vertices": info.processed_vertices,
                "processed_edges": info.processed_edges, "wake_edges": info.wake_edges,
                "device_ms": info.device_ms, "kernel_launches": info.kernel_launches}

    def sync(self):
        import torch
        torch.cuda.synchronize(self.labels.device)

    def free(self):
        if self._h:
            _capi.lib().nulpa_session_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Exchange:
    """The per-pass collectives. `staged=True` runs them on CPU copies (gloo tests)."""

    def __init__(self, bounds: list[int], group=None, staged: bool = False):
        self.bounds = bounds
        self.group = group
        self.staged = staged

    def labels_and_flags(self, labels, flags):
        import torch.distributed as dist
        P = len(self.bounds) - 1
        lab = labels.cpu() if self.staged and labels.is_cuda else labels
        flg = flags.cpu() if self.staged and flags.is_cuda else flags
        # all-gather-v of owned label ranges
        for p in range(P):
            a, b = self.bounds[p], self.bounds[p + 1]
            if b > a:
                dist.broadcast(lab[a:b], src=p, group=self.group)
        # wake flags: MIN-reduce each range to its owner (0 = woken wins)
        for p in range(P):
            a, b = self.bounds[p], self.bounds[p + 1]
            if b > a:
                dist.reduce(flg[a:b], dst=p, op=dist.ReduceOp.MIN, group=self.group)
        if lab is not labels:
            labels.copy_(lab)
            flags.copy_(flg)

    def sum(self, values: list[int]) -> list[int]:
        import torch
        import torch.distributed as dist
        dev = "cpu" if self.staged else f"cuda:{torch.cuda.current_device()}"
        t = torch.tensor(values, dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return [int(round(x)) for x in t.tolist()]


def run_partitioned(engine, cfg: LpaConfig, rank: int, world: int, exchange: Exchange,
                    n: int) -> PartitionedStats:
    """Drive run_engine's schedule (lpa.cpp:270-310) over partitioned passes."""
    import time
    if cfg.cc_period > 0:
        raise ValidationError("cross-check is not supported with a multi-GPU partition")
    if cfg.exec == ExecMode.Sequential:
        raise ValidationError("sequential mode cannot be partitioned across devices")
    lo, hi = exchange.bounds[rank], exchange.bounds[rank + 1]
    st = PartitionedStats()
    engine.init()
    for it in range(cfg.max_iterations):
        pick_less = cfg.pl_period > 0 and it % cfg.pl_period == 0
        was_pl = it > 0 and cfg.pl_period > 0 and (it - 1) % cfg.pl_period == 0
        this_reset = it == 0 or not cfg.prune or (was_pl and not pick_less)
        if not cfg.prune or (was_pl and not pick_less):
            engine.flags.zero_()
        # wake-ups are dead stores when the next pass resets every flag and nothing in
        # this pass can observe them (same rule as run_lpa in engine.cu)
        next_pl = cfg.pl_period > 0 and (it + 1) % cfg.pl_period == 0
        next_reset = it + 1 >= cfg.max_iterations or not cfg.prune or (pick_less and not next_pl)
        wake = not (next_reset and (this_reset or cfg.exec == ExecMode.Synchronous))
        # remote entries: "processed", so only real wake-ups survive the MIN-reduce
        engine.flags[:lo] = 1
        engine.flags[hi:] = 1
        engine.sync()
        info = engine.pass_(pick_less, wake)
        t0 = time.perf_counter()
        exchange.labels_and_flags(engine.labels, engine.flags)
        dn, pe, kl = exchange.sum([info["changed"], info["processed_edges"],
                                   info["kernel_launches"]])
        engine.sync()
        st.exchange_ms.append(1e3 * (time.perf_counter() - t0))
        st.pass_ms.append(info["device_ms"])
        st.processed_edges += pe
        st.kernel_launches += kl
        st.delta_n_per_iter.append(dn)
        st.iterations += 1
        if pick_less:
            st.pl_iterations += 1
        if not pick_less and dn / n < cfg.tolerance:
            st.converged = True
            break
    return st
