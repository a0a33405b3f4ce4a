"""Where the end-to-end (host CSR -> labels) time goes at R-MAT scale s."""
import sys, time, ctypes as C
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2411_11468_b200 import labelprop as lp, _capi
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 27
dg = lp.DeviceGraph.rmat(scale, 16, 1)
n, m2 = dg.n, dg.m2
off_h = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
tgt_h = torch.empty(m2, dtype=torch.int32, pin_memory=True)
lab_h = torch.empty(n, dtype=torch.int32, pin_memory=True)
t0 = time.time()
_capi.check(_capi.lib().nulpa_graph_download(dg._h, off_h.data_ptr(), tgt_h.data_ptr(), None))
print(f"download (vertex order) {time.time()-t0:.3f}s", flush=True)
dg.free()
csr = _capi.nulpa_csr(); csr.n, csr.m2 = n, m2
csr.offsets, csr.targets, csr.weights = off_h.data_ptr(), tgt_h.data_ptr(), None
cfg = lp.LpaConfig()
for rep in range(3):
    t0 = time.time()
    h = C.c_void_p()
    _capi.check(_capi.lib().nulpa_graph_upload(C.byref(csr), 0, C.byref(h)))
    t1 = time.time()
    g = lp.DeviceGraph(h.value, 0)
    o = lp._opts(cfg, 0); st = _capi.nulpa_stats()
    _capi.check(_capi.lib().nulpa_run_graph(g._h, C.byref(o), None, lab_h.data_ptr(), None, C.byref(st)))
    t2 = time.time()
    g.free()
    t3 = time.time()
    print(f"upload+finalize+relayout {t1-t0:.3f}s  run (plan {st.setup_seconds:.3f}s, loop {st.elapsed_seconds:.3f}s, +labels D2H) {t2-t1:.3f}s  free {t3-t2:.3f}s", flush=True)
    st2 = _capi.nulpa_stats()
    t0 = time.time()
    _capi.check(_capi.lib().nulpa_run(C.byref(csr), C.byref(o), None, lab_h.data_ptr(), C.byref(st2)))
    print(f"nulpa_run total {time.time()-t0:.3f}s", flush=True)
