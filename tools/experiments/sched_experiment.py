"""Visit-order experiment: ParallelAsync quality/iterations for ascending vs scrambled order."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import oracle as O
from paper_2411_11468_b200 import labelprop as lp

def sbm(seed):
    g0 = O.RefGraph.planted(100000, 100, 14 / 999, 2 / 99000, seed)
    off, tgt, w = g0.arrays()
    return g0, lp.CsrGraph(off, tgt, w)

for seed in (1,):
    g0, g = sbm(seed)
    qs = O.ref_modularity(g0, O.ref_lpa(g0, exec_mode=2)[0])
    qa = [O.ref_modularity(g0, O.ref_lpa(g0, exec_mode=0, workers=16, switch_degree=0xFFFFFFFF)[0]) for _ in range(3)]
    print(f"SBM seed {seed}: ref sync Q={qs:.4f} ref async16 Q={[round(x,4) for x in qa]}")
    for sched in (1, 2):
        res = []
        for _ in range(3):
            r = lp.lpa(g, lp.LpaConfig(), lp.Tuning(schedule=sched))
            res.append((round(lp.modularity(g, r.labels), 4), r.stats.iterations))
        print(f"   gpu sched={sched}: {res}")
for scale in (20, 24):
    dg = lp.DeviceGraph.rmat(scale, 16, 1)
    for sched in (1, 2):
        for _ in range(2):
            r = dg.lpa(lp.LpaConfig(), lp.Tuning(schedule=sched), want_host=False)
        print(f"rmat{scale} sched={sched}: iters={r.stats.iterations} dn={r.stats.delta_n_per_iter} "
              f"loop={r.stats.elapsed_seconds*1e3:.1f} ms  E/s={dg.m2/r.stats.elapsed_seconds/1e9:.2f}G")
dg = lp.DeviceGraph.grid(4096, 4096)
for sched in (1, 2):
    r = dg.lpa(lp.LpaConfig(), lp.Tuning(schedule=sched), want_host=False)
    r = dg.lpa(lp.LpaConfig(), lp.Tuning(schedule=sched), want_host=False)
    print(f"grid4096 sched={sched}: iters={r.stats.iterations} loop={r.stats.elapsed_seconds*1e3:.1f} ms E/s={dg.m2/r.stats.elapsed_seconds/1e9:.2f}G")
