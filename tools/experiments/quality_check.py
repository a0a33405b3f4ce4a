"""Async quality vs tuning: SBM (n=100K) modularity and R-MAT/grid/web iterations per option.
usage: python tools/quality_check.py key=value ...   (first=0/1 sched=0/1/2)"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2411_11468_b200 import labelprop as lp, workloads
opts = dict(a.split("=") for a in sys.argv[1:])
t = lp.Tuning(async_first_pass=int(opts.get("first", 0)), schedule=int(opts.get("sched", 0)))
for seed in (1, 2, 3):
    dg, _ = workloads.build("sbm", seed=seed)
    g = dg.download()
    qs, its = [], []
    for _ in range(3):
        r = dg.lpa(lp.LpaConfig(), t)
        qs.append(lp.modularity(g, r.labels)); its.append(r.stats.iterations)
    rs = dg.lpa(lp.LpaConfig(exec=lp.ExecMode.Synchronous))
    print(f"{opts} sbm seed {seed}: async Q {np.round(qs, 4).tolist()} iters {its}; "
          f"sync Q {lp.modularity(g, rs.labels):.4f}", flush=True)
for name, dg in (("grid1024", lp.DeviceGraph.grid(1024, 1024)), ("web2M", lp.DeviceGraph.web(2_000_000, 40_000_000, 2.1, 4, 100_000, 1))):
    g = dg.download()
    r = dg.lpa(lp.LpaConfig(), t)
    print(f"{opts} {name}: Q {lp.modularity(g, r.labels):.5f} iters {r.stats.iterations} "
          f"dn {r.stats.delta_n_per_iter}", flush=True)
