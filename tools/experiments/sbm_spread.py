"""Single-run async modularity spread on the smoke/test SBMs vs the reference Synchronous Q."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import oracle as O
from paper_2411_11468_b200 import labelprop as lp
for seed in (1, 2, 3):
    g0 = O.RefGraph.planted(100000, 100, 14 / 999, 2 / 99000, seed)
    off, tgt, w = g0.arrays()
    g = lp.CsrGraph(off, tgt, w)
    pg = O.PortGraph(off, tgt, None)
    lab, _ = O.port_lpa(pg, exec_mode=2)
    qs = O.port_modularity(pg, lab)
    q = [lp.modularity(g, lp.lpa(g).labels) for _ in range(30)]
    print(f"sbm100k seed {seed}: sync {qs:.4f}  async min {min(q):.4f} mean {np.mean(q):.4f} "
          f"max {max(q):.4f}  margin {min(q) - (qs - 0.01):+.4f}", flush=True)
