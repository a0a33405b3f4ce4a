"""Async modularity and iterations, nulpa vs the reference library (oracle/_ref), on the
non-SBM shapes: grid, R-MAT and web-like samples (same CSR arrays for both).
usage: python tools/quality_vs_reference.py"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import oracle as O
from paper_2411_11468_b200 import labelprop as lp

cases = [("grid1024", lambda: lp.DeviceGraph.grid(1024, 1024)),
         ("grid4096", lambda: lp.DeviceGraph.grid(4096, 4096)),
         ("rmat20", lambda: lp.DeviceGraph.rmat(20, 16, 1)),
         ("web2M", lambda: lp.DeviceGraph.web(2_000_000, 40_000_000, 2.1, 4, 100_000, 1))]
for name, mk in cases:
    dg = mk()
    g = dg.download()
    rg = O.RefGraph.from_csr(g.offsets, g.targets, None)
    qs = []
    for _ in range(3):
        r = dg.lpa(lp.LpaConfig())
        qs.append((round(lp.modularity(g, r.labels), 5), r.stats.iterations))
    sw = 32 if int(np.diff(g.offsets).max()) < 32 else 0xFFFFFFFF
    rq = []
    for _ in range(3):
        t = time.time()
        lab, st = O.ref_lpa(rg, exec_mode=0, switch_degree=sw)
        rq.append((round(O.ref_modularity(rg, lab), 5), st["iterations"]))
    ls, ss = O.ref_lpa(rg, exec_mode=2, switch_degree=sw)
    print(f"{name}: n={g.order()} m2={g.directed_size()}  nulpa async (Q, iters) {qs}  "
          f"reference async {rq}  reference sync ({O.ref_modularity(rg, ls):.5f}, "
          f"{ss['iterations']})", flush=True)
