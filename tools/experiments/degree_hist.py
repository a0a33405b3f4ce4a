"""Edge share by degree bucket of the device-built R-MAT graph (tier sizing)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2411_11468_b200 import _capi
from paper_2411_11468_b200 import labelprop as lp
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 27
dg = lp.DeviceGraph.rmat(scale, 16, 1)
off = np.empty(dg.n + 1, np.uint64)
_capi.check(_capi.lib().nulpa_graph_download(dg._h, off.ctypes.data, None, None))
deg = np.diff(off.astype(np.int64))
m2 = deg.sum()
edges = [1, 8, 16, 32, 256, 2048, 8192, 32768, 131072, 524288, 1 << 30]
print(f"scale {scale}: n={dg.n} m2={m2} max_deg={deg.max()} isolated={np.mean(deg == 0):.3f}")
lo = 1
for hi in edges[1:]:
    sel = (deg >= lo) & (deg < hi)
    print(f"  deg [{lo:>7}, {hi:>10}): vertices {sel.sum():>10}  edges {deg[sel].sum() / m2:6.3f}")
    lo = hi
