"""Reference KAT test_lpa.cpp:269-297 (six disjoint dense blocks -> six communities) under
each ParallelAsync schedule, several seeds."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle as O
from paper_2411_11468_b200 import labelprop as lp
for sched in (1, 2, 3):
    res = []
    for seed in (17, 1, 2, 3, 4, 5, 6, 7):
        g0 = O.RefGraph.planted(600, 6, 0.2, 0.0, seed)
        off, tgt, w = g0.arrays()
        g = lp.CsrGraph(off, tgt, w)
        r = lp.lpa(g, lp.LpaConfig(), lp.Tuning(schedule=sched))
        res.append((lp.community_count(g, r.labels), r.stats.converged))
    print("sched", sched, res, flush=True)
