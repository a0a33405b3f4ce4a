"""Reference ParallelAsync on the lattice vs its worker count (the result follows the
workers' contiguous chunks): modularity, iterations, communities."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import oracle as O
from paper_2411_11468_b200 import labelprop as lp
for side in (1024, 4096):
    g = lp.DeviceGraph.grid(side, side).download()
    rg = O.RefGraph.from_csr(g.offsets, g.targets, None)
    for w in (1, 4, 16, 64):
        lab, st = O.ref_lpa(rg, exec_mode=0, workers=w)
        print(f"grid{side} reference async workers={w}: Q {O.ref_modularity(rg, lab):.4f} "
              f"iters {st['iterations']} communities {len(np.unique(lab))}", flush=True)
