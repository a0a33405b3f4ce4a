"""Reproduce the bench's e2e sequence at R-MAT scale s (resident runs, free, host runs)."""
import sys, time, ctypes as C
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2411_11468_b200 import labelprop as lp, _capi
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
resident = len(sys.argv) > 2 and sys.argv[2] == "resident"
dg = lp.DeviceGraph.rmat(scale, 16, 1)
n, m2 = dg.n, dg.m2
cfg = lp.LpaConfig()
if resident:
    for _ in range(3):
        dg.lpa(cfg, lp.Tuning(profile=True), want_host=False)
off_h = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
tgt_h = torch.empty(m2, dtype=torch.int32, pin_memory=True)
lab_h = torch.empty(n, dtype=torch.int32, pin_memory=True)
_capi.check(_capi.lib().nulpa_graph_download(dg._h, off_h.data_ptr(), tgt_h.data_ptr(), None))
ref = dg.lpa(lp.LpaConfig(exec=lp.ExecMode.Synchronous, max_iterations=2)).labels if scale <= 22 else None
dg.free()
csr = _capi.nulpa_csr(); csr.n, csr.m2 = n, m2
csr.offsets, csr.targets, csr.weights = off_h.data_ptr(), tgt_h.data_ptr(), None
o = lp._opts(cfg, 0)
for rep in range(3):
    st = _capi.nulpa_stats()
    t0 = time.time()
    rc = _capi.lib().nulpa_run(C.byref(csr), C.byref(o), None, lab_h.data_ptr(), C.byref(st))
    print(f"scale {scale} rep {rep}: rc {rc} {time.time()-t0:.3f}s loop {st.elapsed_seconds:.3f} iters {st.iterations}", flush=True)
    if rc:
        print(_capi.lib().nulpa_last_error()); break
if ref is not None:
    o2 = lp._opts(lp.LpaConfig(exec=lp.ExecMode.Synchronous, max_iterations=2), 0)
    st = _capi.nulpa_stats()
    _capi.check(_capi.lib().nulpa_run(C.byref(csr), C.byref(o2), None, lab_h.data_ptr(), C.byref(st)))
    print("sync labels equal:", np.array_equal(lab_h.numpy().view(np.uint32), ref))
