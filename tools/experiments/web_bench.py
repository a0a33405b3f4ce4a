"""Per-tier timing on the web-like workload (50M vertices, ~1B draws, 16 hubs of ~2M)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import ctypes as C, numpy as np
from paper_2411_11468_b200 import labelprop as lp, _capi, workloads
dg, _ = workloads.build("web")
cfg = lp.LpaConfig(); t = lp.Tuning(profile=True)
for _ in range(2): dg.lpa(cfg, t, want_host=False)
r = dg.lpa(cfg, t, want_host=False)
o = lp._opts(cfg, 0); st = _capi.nulpa_stats(); tc = t.to_c()
_capi.check(_capi.lib().nulpa_run_graph(dg._h, C.byref(o), C.byref(tc), None, None, C.byref(st)))
print(f"web loop {st.elapsed_seconds*1e3:.1f} ms iters {st.iterations} -> {dg.m2/st.elapsed_seconds/1e9:.2f} G edges/s")
print("tiers ms:", {n: round(st.tier_ms[i], 2) for i, n in enumerate(_capi.TIER_NAMES) if st.tier_ms[i]})
