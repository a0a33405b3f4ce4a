"""Quick per-tier timing: build R-MAT (or another workload) on the device, warm up, time lpa().
usage: python tools/tier_bench.py [scale] [reps]"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_11468_b200 import labelprop as lp, _capi
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 27
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
t0 = time.time()
dg = lp.DeviceGraph.rmat(scale, 16, 1)
print(f"scale {scale}: n={dg.n} m2={dg.m2} build {time.time()-t0:.2f}s", flush=True)
cfg = lp.LpaConfig()
opts = dict(a.split("=") for a in sys.argv[3:])
if "iters" in opts:
    cfg = lp.LpaConfig(max_iterations=int(opts["iters"]))
t = lp.Tuning(profile=True, async_first_pass=int(opts.get("first", 0)),
              schedule=int(opts.get("sched", 0)), thread_max_degree=int(opts.get("tmax", 0)),
              warp_max_degree=int(opts.get("wmax", 0)), block_max_degree=int(opts.get("bmax", 0)))
if opts.get("workload") == "sbm":
    pass
for _ in range(2):
    dg.lpa(cfg, t, want_host=False)
import ctypes as C, numpy as np
tot = np.zeros(_capi.NULPA_TIERS); loop = 0.0
for _ in range(reps):
    o = lp._opts(cfg, 0)
    st = _capi.nulpa_stats()
    dn = np.zeros(20, np.uint64); st.delta_n = dn.ctypes.data_as(C.POINTER(C.c_uint64))
    tc = t.to_c()
    _capi.check(_capi.lib().nulpa_run_graph(dg._h, C.byref(o), C.byref(tc), None, None, C.byref(st)))
    tot += np.array([st.tier_ms[i] for i in range(_capi.NULPA_TIERS)]); loop += st.elapsed_seconds
    edges = [st.tier_edges[i] for i in range(_capi.NULPA_TIERS)]
print(f"{opts} loop {loop/reps*1e3:.1f} ms  iters {st.iterations} dn {dn[:st.iterations].tolist()} "
      f"-> {dg.m2/(loop/reps)/1e9:.2f} G edges/s")
print("tiers ms:", {n: round(x / reps, 2) for n, x in zip(_capi.TIER_NAMES, tot) if x})
print("tier edges (last run):", {n: x for n, x in zip(_capi.TIER_NAMES, edges) if x})
