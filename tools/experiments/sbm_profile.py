import sys, ctypes as C
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_2411_11468_b200 import labelprop as lp, workloads, _capi
dg, _ = workloads.build("sbm", seed=1)
cfg = lp.LpaConfig()
for prof in (False, True, False):
    t = lp.Tuning(profile=prof)
    for _ in range(3):
        o = lp._opts(cfg, 0); st = _capi.nulpa_stats(); tc = t.to_c()
        _capi.check(_capi.lib().nulpa_run_graph(dg._h, C.byref(o), C.byref(tc), None, None, C.byref(st)))
    tiers = [st.tier_ms[i] for i in range(_capi.NULPA_TIERS)]
    print(f"profile={prof} loop {st.elapsed_seconds*1e3:.3f} ms iters {st.iterations} launches {st.kernel_launches} tier ms sum {sum(tiers):.3f} {[round(x,3) for x in tiers]}")
