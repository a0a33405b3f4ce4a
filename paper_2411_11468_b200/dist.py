"""Partitioned multi-GPU ν-LPA: one process per GPU, torch.distributed plumbing.

Layout: a 1-D edge-balanced partition of the resident position order (rank p owns
positions [b_p, b_{p+1}) with offsets[b_p] ~ p*m2/P, `nulpa_graph_edge_ranges`). Each rank
keeps ONLY its rows on the device (`nulpa_graph_slice`: targets are global position ids);
labels u32[n] and wake flags u8[n] are replicated on every rank, in position order
(`DeviceRangeEngine.vertex_labels` returns vertex order). Each pass:

1. every rank runs one pass over its own rows (`nulpa_session_pass`, kernels on the
   collective stream): ParallelAsync in place inside the range, Synchronous into a
   staging buffer then applied; neighbour wake-ups write flags[j] = 0 for owned AND
   remote j;
2. counters (changed, processed vertices / edges / wakes, launches): one all-gather of
   a P x 6 tensor — the pass's only host read (run_engine needs dN on the host to test
   convergence, lpa.cpp:306);
3. labels: if the largest per-rank change count is small, the changed-only exchange —
   each rank packs its (position, label) pairs (`nulpa_session_pack_changes`), one
   all-gather of the padded packets, each rank applies them — else one all-gather of the
   owned ranges padded to the longest range;
4. wake flags: remote entries were primed to 1 ("processed") before the pass, so one
   MIN reduce-scatter of the padded flag ranges delivers every rank's wake-ups of the
   vertices it owns (0 = woken wins).

Everything is issued on one CUDA stream (the session runs on torch's current stream), so
the only synchronisation per pass is the counter read. The run_engine schedule
(lpa.cpp:246-315: Pick-Less every pl_period, flag reset on leaving a PL pass or without
pruning, dN/n < tolerance on a non-PL pass) is driven on the host, identically on every
rank. Across ranks the passes are Jacobi (remote labels are one pass stale); a
Synchronous run is therefore bit-identical to the single-GPU Synchronous run.
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
    exchange_bytes: list[int] = field(default_factory=list)  # bytes this rank contributed
    exchange_modes: list[str] = field(default_factory=list)
    processed_vertices: int = 0     # all ranks
    processed_edges: int = 0        # all ranks
    wake_edges: int = 0             # all ranks
    changed: int = 0                # all ranks
    local_bytes: float = 0.0        # this rank's algorithmic bytes
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
    """One rank's pass engine: a nulpa_session over its rows of a DeviceGraph, on torch
    tensors. With `own_rows_only` the session runs on a slice of the graph that holds just
    the rank's rows (nulpa_graph_slice); the full graph may then be freed."""

    def __init__(self, dg, cfg: LpaConfig, lo: int, hi: int, tuning: Tuning | None = None,
                 own_rows_only: bool = False):
        import torch
        self.n = dg.n
        self.lo, self.hi = lo, hi
        self.device = dg.device
        dev = f"cuda:{dg.device}"
        if own_rows_only:
            from .labelprop import DeviceGraph
            h = C.c_void_p()
            _capi.check(_capi.lib().nulpa_graph_slice(dg._h, lo, hi, C.byref(h)))
            self.graph = DeviceGraph(h.value, dg.device)
        else:
            self.graph = dg
        self.labels = torch.empty(dg.n, dtype=torch.int32, device=dev)
        self.flags = torch.empty(dg.n, dtype=torch.uint8, device=dev)
        o = _opts(cfg, dg.device)
        t = tuning.to_c() if tuning else None
        h = C.c_void_p()
        _capi.check(_capi.lib().nulpa_session_create(self.graph._h, C.byref(o),
                                                     C.byref(t) if t else None, lo, hi,
                                                     self.labels.data_ptr(),
                                                     self.flags.data_ptr(), C.byref(h)))
        self._h = h
        # the session's kernels run on the stream the collectives use
        _capi.check(_capi.lib().nulpa_session_set_stream(
            self._h, C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)))

    def init(self):
        _capi.check(_capi.lib().nulpa_session_init(self._h))

    def vertex_labels(self):
        """The replicated labels (position order inside the session) in vertex order."""
        import torch
        out = torch.empty_like(self.labels)
        self.graph.labels_to_vertex_order(self.labels.data_ptr(), out.data_ptr())
        return out

    def pass_(self, pick_less: bool, wake: bool = True) -> dict:
        info = _capi.nulpa_pass_info()
        _capi.check(_capi.lib().nulpa_session_pass(self._h, int(pick_less), int(wake),
                                                   C.byref(info)))
        return {"changed": info.changed, "processed_vertices": info.processed_vertices,
                "processed_edges": info.processed_edges, "wake_edges": info.wake_edges,
                "device_ms": info.device_ms, "kernel_launches": info.kernel_launches}

    def pack_changes(self, out, cap: int) -> None:
        import torch
        _capi.check(_capi.lib().nulpa_session_pack_changes(
            self._h, C.c_void_p(out.data_ptr()), cap,
            C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)))

    def apply_changes(self, packets, pairs: int) -> None:
        import torch
        _capi.check(_capi.lib().nulpa_session_apply_changes(
            self._h, C.c_void_p(packets.data_ptr()), pairs,
            C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)))

    def community_sums(self):
        """sigma_c and Sigma_c (n doubles each, indexed by label) over this rank's rows
        (quality.cpp:29-40); summed over the ranks they give the graph's modularity."""
        import torch
        sig = torch.empty(self.n, dtype=torch.float64, device=self.labels.device)
        big = torch.empty_like(sig)
        _capi.check(_capi.lib().nulpa_community_sums_graph(
            self.graph._h, C.c_void_p(self.labels.data_ptr()), C.c_void_p(sig.data_ptr()),
            C.c_void_p(big.data_ptr())))
        return sig, big

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
    """The per-pass collectives over padded ranges (module docstring, steps 2-4).
    `staged=True` runs them on CPU copies through gloo (the CPU tests; gloo has no
    reduce-scatter, so the flags there use an all-reduce)."""

    def __init__(self, bounds: list[int], group=None, staged: bool = False,
                 changed_only: bool = True):
        self.bounds = bounds
        self.group = group
        self.staged = staged
        self.changed_only = changed_only
        self.P = len(bounds) - 1
        self.L = max(1, max(b - a for a, b in zip(bounds, bounds[1:])))

    def _coll(self, t):
        return t.cpu() if self.staged and t.is_cuda else t

    def counters(self, values: list[int]) -> np.ndarray:
        """All ranks' counters, P x len(values) (one all-gather, one host read)."""
        import torch
        import torch.distributed as dist
        dev = "cpu" if self.staged else f"cuda:{torch.cuda.current_device()}"
        t = torch.tensor(values, dtype=torch.int64, device=dev)
        out = torch.empty(self.P * len(values), dtype=torch.int64, device=dev)
        if self.staged:
            parts = list(out.chunk(self.P))
            dist.all_gather(parts, t, group=self.group)
            out = torch.cat(parts)
        else:
            dist.all_gather_into_tensor(out, t, group=self.group)
        return out.cpu().numpy().reshape(self.P, len(values))

    def labels(self, engine, rank: int, max_changed: int) -> tuple[str, int]:
        """Bring every replica's labels up to date; returns (mode, bytes sent)."""
        import torch
        import torch.distributed as dist
        lab = engine.labels
        if self.changed_only and 2 * max_changed < self.L:
            cap = max(1, max_changed)
            mine = torch.empty(2 * cap, dtype=torch.int32, device=lab.device)
            engine.pack_changes(mine, cap)
            allp = self._gather(mine)
            if self.staged:
                allp = allp.to(lab.device)
            engine.apply_changes(allp, self.P * cap)
            return "changed-only", 8 * cap
        a, b = self.bounds[rank], self.bounds[rank + 1]
        send = torch.zeros(self.L, dtype=torch.int32, device=lab.device)
        send[:b - a] = lab[a:b]
        recv = self._gather(send)
        for q in range(self.P):
            if q != rank:
                qa, qb = self.bounds[q], self.bounds[q + 1]
                lab[qa:qb] = recv[q * self.L:q * self.L + qb - qa].to(lab.device)
        return "full", 4 * self.L

    def _gather(self, t):
        import torch
        import torch.distributed as dist
        src = self._coll(t)
        if self.staged:
            parts = [torch.empty_like(src) for _ in range(self.P)]
            dist.all_gather(parts, src, group=self.group)
            return torch.cat(parts)
        out = torch.empty(self.P * src.numel(), dtype=src.dtype, device=src.device)
        dist.all_gather_into_tensor(out, src, group=self.group)
        return out

    def flags(self, engine, rank: int) -> int:
        """MIN-reduce every rank's view of each owner's flag range into the owner."""
        import torch
        import torch.distributed as dist
        flg = engine.flags
        buf = torch.ones(self.P * self.L, dtype=torch.uint8, device=flg.device)
        for q in range(self.P):
            qa, qb = self.bounds[q], self.bounds[q + 1]
            buf[q * self.L:q * self.L + qb - qa] = flg[qa:qb]
        a, b = self.bounds[rank], self.bounds[rank + 1]
        if self.staged:
            cb = buf.cpu()
            dist.all_reduce(cb, op=dist.ReduceOp.MIN, group=self.group)
            mine = cb[rank * self.L:rank * self.L + b - a].to(flg.device)
        else:
            out = torch.empty(self.L, dtype=torch.uint8, device=flg.device)
            dist.reduce_scatter_tensor(out, buf, op=dist.ReduceOp.MIN, group=self.group)
            mine = out[:b - a]
        flg[a:b] = mine
        return self.P * self.L


def pass_bytes(info: dict, list_len: int, weighted: bool = False) -> float:
    """SURVEY §8d algorithmic bytes of one rank's pass (flag sweep, row bounds + own
    label, target + neighbour label per scanned edge, label writes, wake stores)."""
    return (list_len + 12.0 * info["processed_vertices"]
            + (12.0 if weighted else 8.0) * info["processed_edges"]
            + 4.0 * info["changed"] + 1.0 * info["wake_edges"])


def run_partitioned(engine, cfg: LpaConfig, rank: int, world: int, exchange: Exchange,
                    n: int) -> PartitionedStats:
    """Drive run_engine's schedule (lpa.cpp:270-310) over partitioned passes."""
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
        info = engine.pass_(pick_less, wake)
        cnt = exchange.counters([info["changed"], info["processed_vertices"],
                                 info["processed_edges"], info["wake_edges"],
                                 info["kernel_launches"], 0])
        dn = int(cnt[:, 0].sum())
        mode, nbytes = exchange.labels(engine, rank, int(cnt[:, 0].max()))
        if wake:
            nbytes += exchange.flags(engine, rank)
        st.exchange_modes.append(mode)
        st.exchange_bytes.append(nbytes)
        st.pass_ms.append(info["device_ms"])
        st.processed_vertices += int(cnt[:, 1].sum())
        st.processed_edges += int(cnt[:, 2].sum())
        st.wake_edges += int(cnt[:, 3].sum())
        st.changed += dn
        st.kernel_launches += int(cnt[:, 4].sum())
        st.local_bytes += pass_bytes(info, hi - lo)
        st.delta_n_per_iter.append(dn)
        st.iterations += 1
        if pick_less:
            st.pl_iterations += 1
        if not pick_less and dn / n < cfg.tolerance:
            st.converged = True
            break
    return st


def partitioned_modularity(engine, group=None, staged: bool = False) -> float:
    """The graph's modularity (quality.cpp:21-49) from the ranks' row slices: sigma_c and
    Sigma_c summed over ranks (one all-reduce), then folded on every rank."""
    import torch
    import torch.distributed as dist
    sig, big = engine.community_sums()
    both = torch.stack([sig, big])
    if staged:
        cb = both.cpu()
        dist.all_reduce(cb, group=group)
        both = cb.to(sig.device)
    else:
        dist.all_reduce(both, group=group)
    sig, big = both[0], both[1]
    two_m = float(big.sum())
    return float((sig / two_m - (big / two_m) ** 2).sum())
