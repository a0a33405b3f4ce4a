"""Wide-tier work model on the device-built R-MAT graph: rows with 6144 < d <= 98304,
their edges and the label-partitioned phase count P = ceil(d / 12288) of a first pass."""
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
for lo, hi in [(1025, 6144), (6145, 98304), (98305, 1 << 40)]:
    sel = (deg >= lo) & (deg <= hi)
    d = deg[sel]
    print(f"deg [{lo}, {hi}]: rows {d.size} edges {d.sum()} ({d.sum() / m2:.3f} of m2)")
d = deg[(deg > 6144) & (deg <= 98304)]
for lim in (6144, 12288, 24576):
    P = (d + lim - 1) // lim
    print(f"  limit {lim}: rows with P>1 {np.sum(P > 1)}  edges in P>1 rows {d[P > 1].sum()}  "
          f"sum P*d {np.sum(P * d)}  ratio {np.sum(P * d) / d.sum():.2f}")
