import sys; sys.path.insert(0, '/root/repo')
import numpy as np
from paper_2411_11468_b200 import labelprop as lp
d = dict(np.load('/root/repo/tests/golden/sbm10k_seed101.npz'))
g = lp.CsrGraph(d["offsets"], d["targets"], d["weights"])
qs = [lp.modularity(g, lp.lpa(g).labels) for _ in range(40)]
print(f"min {min(qs):.4f} mean {np.mean(qs):.4f} max {max(qs):.4f}")
