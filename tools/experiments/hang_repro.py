"""Replays the tail of bench.py's default run step by step with timestamps (the default
bench stalled after the reference modularity on the box)."""
import faulthandler
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
faulthandler.dump_traceback_later(240, repeat=True)
import torch  # noqa: E402

import oracle as O  # noqa: E402
from paper_2411_11468_b200 import labelprop as lp  # noqa: E402

t0 = time.time()


def log(m):
    print(f"[{time.time() - t0:7.1f}] {m}", flush=True)


big = sys.argv[1] == "big" if len(sys.argv) > 1 else True
if big:
    dg = lp.DeviceGraph.rmat(27, 16, 1)
    off_h = torch.empty(dg.n + 1, dtype=torch.int64, pin_memory=True)
    tgt_h = torch.empty(dg.m2, dtype=torch.int32, pin_memory=True)
    log("pinned allocated")
    dg.free()
sg = O.RefGraph.planted(100000, 100, 14 / 999, 2 / 99000, 1)
so, st_, _ = sg.arrays()
sgh = lp.CsrGraph(so, st_, None)
log("sbm built")
for k in range(5):
    r = lp.lpa(sgh)
    log(f"nulpa lpa {k}: {r.stats.iterations} iters")
    q = lp.modularity(sgh, r.labels)
    log(f"nulpa modularity {q:.4f}")
import bench  # noqa: E402
out = bench.sbm_quality([q])
log(f"sbm_quality done {out['ref_sync_Q']:.4f} {out['ref_async_Q']}")
