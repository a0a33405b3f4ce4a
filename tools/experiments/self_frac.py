"""Fraction of edge endpoints whose label equals their own vertex id after k passes,
per degree tier of the row owner (R-MAT scale s)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2411_11468_b200 import labelprop as lp
s = int(sys.argv[1]) if len(sys.argv) > 1 else 22
dg = lp.DeviceGraph.rmat(s, 16, 1)
g = dg.download()
off = g.offsets.astype(np.int64); tgt = g.targets.astype(np.int64)
deg = np.diff(off)
src = np.repeat(np.arange(g.order()), deg)
bounds = [(1, 32), (33, 256), (257, 1024), (1025, 4096), (4097, 12288), (12289, 98304), (98305, 1 << 40)]
for k in (1, 2):
    lab = dg.lpa(lp.LpaConfig(max_iterations=k)).labels.astype(np.int64)
    selfl = lab[tgt] == tgt
    out = []
    for lo, hi in bounds:
        m = (deg[src] >= lo) & (deg[src] <= hi)
        if m.any():
            # distinct non-self labels per row vs row length
            out.append(f"{lo}-{hi}: self {selfl[m].mean():.2f}")
    print(f"after {k} pass(es):", "; ".join(out), flush=True)
