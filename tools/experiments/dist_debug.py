"""Single-process emulation of the 2-rank partitioned Synchronous run (dist.py) on one GPU:
two sessions, the exchange done with plain tensor copies. Prints dN per pass against the
single-GPU Synchronous run, with and without row slices (own_rows_only)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import ctypes as C  # noqa: E402

import torch  # noqa: E402

from paper_2411_11468_b200 import _capi  # noqa: E402
from paper_2411_11468_b200 import labelprop as lp  # noqa: E402
from paper_2411_11468_b200.dist import DeviceRangeEngine  # noqa: E402
from paper_2411_11468_b200.labelprop import ExecMode, LpaConfig  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 14
mode = sys.argv[2] if len(sys.argv) > 2 else "sync"
cfg = LpaConfig(exec=ExecMode.Synchronous if mode == "sync" else ExecMode.ParallelAsync)
dg = lp.DeviceGraph.rmat(scale, 16, 5)
want = dg.lpa(cfg)
print("single:", want.stats.delta_n_per_iter)
P = 2
b = (C.c_uint32 * (P + 1))()
_capi.check(_capi.lib().nulpa_graph_edge_ranges(dg._h, P, b))
bounds = list(b)
print("bounds", bounds)
for own in (False, True):
    engs = [DeviceRangeEngine(dg, cfg, bounds[r], bounds[r + 1], own_rows_only=own) for r in range(P)]
    for e in engs:
        e.init()
    dns = []
    for it in range(cfg.max_iterations):
        pl = cfg.pl_period > 0 and it % cfg.pl_period == 0
        was_pl = it > 0 and cfg.pl_period > 0 and (it - 1) % cfg.pl_period == 0
        if not cfg.prune or (was_pl and not pl):
            for e in engs:
                e.flags.zero_()
        for r, e in enumerate(engs):
            e.flags[:bounds[r]] = 1
            e.flags[bounds[r + 1]:] = 1
        infos = [e.pass_(pl, True) for e in engs]
        torch.cuda.synchronize()
        dn = sum(i["changed"] for i in infos)
        # labels: owner ranges to every replica
        for r, e in enumerate(engs):
            for q, f in enumerate(engs):
                if q != r:
                    f.labels[bounds[r]:bounds[r + 1]] = e.labels[bounds[r]:bounds[r + 1]]
        # flags: MIN over replicas into the owner
        for r, e in enumerate(engs):
            m = torch.stack([f.flags[bounds[r]:bounds[r + 1]] for f in engs]).min(0).values
            e.flags[bounds[r]:bounds[r + 1]] = m
        torch.cuda.synchronize()
        dns.append(dn)
        if not pl and dn / dg.n < cfg.tolerance:
            break
    lab = engs[0].vertex_labels().cpu().numpy().view(np.uint32)
    print(f"own_rows_only={own}: {dns} labels equal: {np.array_equal(lab, want.labels)}",
          "mismatch", int((lab != want.labels).sum()))
    for e in engs:
        e.free()

# ---- pass-0 detail: per-rank changes and the slice's rows against the full graph's
full = dg.download()
for r in range(P):
    lo, hi = bounds[r], bounds[r + 1]
    ea = DeviceRangeEngine(dg, cfg, lo, hi, own_rows_only=False)
    eb = DeviceRangeEngine(dg, cfg, lo, hi, own_rows_only=True)
    so = np.empty(dg.n + 1, np.uint64)
    st = np.empty(max(1, eb.graph.m2), np.uint32)
    _capi.check(_capi.lib().nulpa_graph_download_raw(eb.graph._h, so.ctypes.data, st.ctypes.data, None))
    fo = np.empty(dg.n + 1, np.uint64)
    ft = np.empty(dg.m2, np.uint32)
    _capi.check(_capi.lib().nulpa_graph_download_raw(dg._h, fo.ctypes.data, ft.ctypes.data, None))
    rows_ok = all(np.array_equal(ft[fo[v]:fo[v + 1]], st[so[v]:so[v + 1]]) for v in range(lo, hi))
    print(f"rank {r} [{lo},{hi}) slice m2={eb.graph.m2} rows equal: {rows_ok}; "
          f"slice max_degree/rows_simple via pass:")
    for e in (ea, eb):
        e.init()
        info = e.pass_(True, True)
        torch.cuda.synchronize()
        print("   ", "slice" if e is eb else "full ", info)
    la = ea.labels.cpu().numpy().view(np.uint32)
    lb = eb.labels.cpu().numpy().view(np.uint32)
    diff = np.nonzero(la != lb)[0]
    print("    differing positions:", diff[:10], len(diff))
    for p in diff[:3]:
        print("     pos", p, "full", la[p], "slice", lb[p], "deg", int(fo[p + 1] - fo[p]),
              "row", ft[fo[p]:fo[p + 1]][:8])
    ea.free()
    eb.free()
