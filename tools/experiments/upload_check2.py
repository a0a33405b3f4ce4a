import sys, os
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2411_11468_b200 import labelprop as lp
for scale in (16, 18, 19, 20):
    for chunk in (None, "100000"):
        if chunk: os.environ["NULPA_UPLOAD_CHUNK"] = chunk
        else: os.environ.pop("NULPA_UPLOAD_CHUNK", None)
        dg = lp.DeviceGraph.rmat(scale, 16, 1)
        g = dg.download()
        up = lp.DeviceGraph.upload(lp.CsrGraph(g.offsets, g.targets, None))
        h = up.download()
        bad = np.flatnonzero(h.targets != g.targets)
        deg = np.diff(g.offsets.astype(np.int64))
        rows = np.searchsorted(g.offsets.astype(np.int64), bad, side="right") - 1 if bad.size else []
        print(f"scale {scale} chunk {chunk}: mismatches {bad.size}; rows {len(set(rows.tolist())) if bad.size else 0}; "
              f"degrees {sorted(set(deg[rows].tolist()))[:10] if bad.size else []}", flush=True)
