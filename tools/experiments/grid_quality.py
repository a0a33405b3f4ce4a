"""Grid (lattice) async quality vs the visit order: Q and iterations per schedule."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_11468_b200 import labelprop as lp
for side in (1024, 4096):
    dg = lp.DeviceGraph.grid(side, side)
    g = dg.download()
    for sched in (4,):
        out = []
        for _ in range(2):
            r = dg.lpa(lp.LpaConfig(), lp.Tuning(schedule=sched))
            out.append((round(lp.modularity(g, r.labels), 4), r.stats.iterations,
                        lp.community_count(g, r.labels)))
        print(f"grid{side} schedule {sched}: (Q, iters, communities) {out}", flush=True)
