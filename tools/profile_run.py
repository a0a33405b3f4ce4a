"""Workload for ncu captures: build a bench workload on the device, warm up, run lpa().
    python tools/profile_run.py [SCALE|WORKLOAD] [SCHEDULE] [RUNS]
SCALE = an R-MAT scale (default 24); WORKLOAD = rmat | grid | web | sbm (bench.py's)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_11468_b200 import labelprop as lp  # noqa: E402
from paper_2411_11468_b200 import workloads  # noqa: E402
arg = sys.argv[1] if len(sys.argv) > 1 else "24"
sched = int(sys.argv[2]) if len(sys.argv) > 2 else 0
runs = int(sys.argv[3]) if len(sys.argv) > 3 else 2
if arg.isdigit():
    dg = lp.DeviceGraph.rmat(int(arg), 16, 1)
else:
    dg, _ = workloads.build(arg)
for _ in range(runs):
    r = dg.lpa(lp.LpaConfig(), lp.Tuning(schedule=sched), want_host=False)
print(r.stats.iterations, r.stats.elapsed_seconds)
