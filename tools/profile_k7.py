"""Workload for the K7 ncu capture: one lpa() run on a device R-MAT graph, then modularity."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from paper_2411_11468_b200 import labelprop as lp  # noqa: E402
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
dg = lp.DeviceGraph.rmat(scale, 16, 1)
lab = torch.empty(dg.n, dtype=torch.int32, device="cuda:0")
dg.lpa(lp.LpaConfig(), labels_device_ptr=lab.data_ptr(), want_host=False)
print(dg.modularity_device(lab.data_ptr()))
