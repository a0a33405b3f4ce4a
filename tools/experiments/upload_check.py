"""Pipelined upload vs device-built graph at R-MAT scale s: CSR equality and Synchronous runs."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2411_11468_b200 import labelprop as lp
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
dg = lp.DeviceGraph.rmat(scale, 16, 1)
g = dg.download()
up = lp.DeviceGraph.upload(lp.CsrGraph(g.offsets, g.targets, None))
h = up.download()
print("offsets equal", np.array_equal(h.offsets, g.offsets), "targets equal", np.array_equal(h.targets, g.targets))
print("max_degree", dg.max_degree, up.max_degree)
for first in (True, False):
    t = lp.Tuning(identity_first=first)
    for it in (1, 2, 3):
        a = dg.lpa(lp.LpaConfig(exec=lp.ExecMode.Synchronous, max_iterations=it), t)
        b = up.lpa(lp.LpaConfig(exec=lp.ExecMode.Synchronous, max_iterations=it), t)
        print(f"identity_first={first} iters={it}: equal {np.array_equal(a.labels, b.labels)} dn {a.stats.delta_n_per_iter} {b.stats.delta_n_per_iter}")
