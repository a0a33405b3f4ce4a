"""Wall time of nulpa_run_graph vs its loop time (resident R-MAT), with/without profiling."""
import sys, time, ctypes as C
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2411_11468_b200 import labelprop as lp, _capi
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 27
dg = lp.DeviceGraph.rmat(scale, 16, 1)
cfg = lp.LpaConfig()
for prof in (0, 1, 0):
    t = lp.Tuning(profile=bool(prof)).to_c()
    for rep in range(4):
        o = lp._opts(cfg, 0); st = _capi.nulpa_stats()
        t0 = time.perf_counter()
        _capi.check(_capi.lib().nulpa_run_graph(dg._h, C.byref(o), C.byref(t), None, None, C.byref(st)))
        w = time.perf_counter() - t0
        print(f"profile={prof} wall {w*1e3:.1f} ms loop {st.elapsed_seconds*1e3:.1f} setup {st.setup_seconds*1e3:.1f}", flush=True)
