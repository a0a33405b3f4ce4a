import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2411_11468_b200 import labelprop as lp
scale = int(sys.argv[1])
dg = lp.DeviceGraph.rmat(scale, 16, 1)
g = dg.download()
dg.free()
up = lp.DeviceGraph.upload(lp.CsrGraph(g.offsets, g.targets, None))
print("uploaded", up.n, up.m2, up.max_degree, flush=True)
