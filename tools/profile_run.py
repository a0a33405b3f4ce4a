"""Workload for ncu captures: build R-MAT on the device, warm up, run one lpa()."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_11468_b200 import labelprop as lp
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
sched = int(sys.argv[2]) if len(sys.argv) > 2 else 0
dg = lp.DeviceGraph.rmat(scale, 16, 1)
runs = int(sys.argv[3]) if len(sys.argv) > 3 else 2
for _ in range(runs):
    r = dg.lpa(lp.LpaConfig(), lp.Tuning(schedule=sched), want_host=False)
print(r.stats.iterations, r.stats.elapsed_seconds)
