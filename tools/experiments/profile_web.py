import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_11468_b200 import labelprop as lp, workloads
dg, _ = workloads.build("web")
r = dg.lpa(lp.LpaConfig(), want_host=False)
print(r.stats.iterations)
