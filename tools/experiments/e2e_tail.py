"""Time the tail of nulpa_run_graph (labels to vertex order + D2H) at R-MAT scale s."""
import sys, time, ctypes as C
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2411_11468_b200 import labelprop as lp, _capi
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 27
dg = lp.DeviceGraph.rmat(scale, 16, 1)
n = dg.n
lab_h = torch.empty(n, dtype=torch.int32, pin_memory=True)
lab_d = torch.empty(n, dtype=torch.int32, device="cuda:0")
cfg = lp.LpaConfig()
o = lp._opts(cfg, 0)
for mode in ("none", "device", "host", "none", "host", "device"):
    st = _capi.nulpa_stats()
    torch.cuda.synchronize()
    t0 = time.time()
    _capi.check(_capi.lib().nulpa_run_graph(
        dg._h, C.byref(o), None, lab_h.data_ptr() if mode == "host" else None,
        lab_d.data_ptr() if mode == "device" else None, C.byref(st)))
    torch.cuda.synchronize()
    t = time.time() - t0
    print(f"{mode:6s} total {t:.3f}s setup {st.setup_seconds:.3f}s loop {st.elapsed_seconds:.3f}s "
          f"tail {t - st.setup_seconds - st.elapsed_seconds:.3f}s", flush=True)
