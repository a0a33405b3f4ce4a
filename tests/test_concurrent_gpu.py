"""Side-by-side tier groups (NULPA_CONCURRENT) and the one-step-at-a-time semantics of the
batched warp tiers (NULPA_GROUP_STEPS with intra-chunk patching).

Each configuration runs in a child process (the switches are read once per process):
- Synchronous runs are a pure function of the graph (lpa.cpp:70-100), so every tier
  schedule must give the same labels and ΔN trajectory bit for bit;
- ParallelAsync runs must converge with the quality bar of the SBM-100K gate
  (reference Synchronous Q 0.843032 - 0.01, SURVEY §8c gate 3) and keep the reference's
  star KAT (test_lpa.cpp:256-267: the low list before the team list).
"""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

CHILD = r"""
import hashlib, json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2411_11468_b200 import labelprop as lp, workloads
out = {}
for scale in (12, 16):
    dg = lp.DeviceGraph.rmat(scale, 16, seed=5)
    r = dg.lpa(lp.LpaConfig(exec=lp.ExecMode.Synchronous))
    out[f"sync{scale}"] = [hashlib.sha1(r.labels.tobytes()).hexdigest(),
                           r.stats.delta_n_per_iter]
dg, _ = workloads.build("sbm", seed=1)
g = dg.download()
qs = []
for _ in range(3):
    r = dg.lpa(lp.LpaConfig())
    qs.append(lp.modularity(g, r.labels))
out["sbm_q"] = qs
# star(40) with switch_degree 8 (hub on the team path), pl_period 0
u = np.zeros(40, np.uint32); v = np.arange(1, 41, dtype=np.uint32)
sg = lp.DeviceGraph.from_edges(u, v, 41)
r = sg.lpa(lp.LpaConfig(switch_degree=8, pl_period=0))
out["star"] = [r.labels.tolist(), r.stats.delta_n_per_iter]
print(json.dumps(out))
"""


def run_child(**env):
    e = dict(os.environ)
    e.update({k: str(v) for k, v in env.items()})
    p = subprocess.run([sys.executable, "-c", CHILD, str(ROOT)], env=e, capture_output=True,
                       text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


@pytest.fixture(scope="module")
def serial():
    return run_child(NULPA_CONCURRENT=0, NULPA_GROUP_STEPS=1)


@pytest.mark.parametrize("env", [
    {"NULPA_CONCURRENT": 1},
    {"NULPA_CONCURRENT": 2},
    {"NULPA_CONCURRENT": 3},
    {"NULPA_CONCURRENT": 2, "NULPA_GROUP_STEPS": 1},
    {"NULPA_CONCURRENT": 2, "NULPA_GROUP_STEPS": 8},
    {"NULPA_CONCURRENT": 2, "NULPA_SMALL_TIER_BATCH": 0},
])
def test_tier_schedules(serial, env):
    got = run_child(**env)
    for scale in (12, 16):
        assert got[f"sync{scale}"] == serial[f"sync{scale}"], f"Synchronous differs at R-MAT {scale}"
    assert min(got["sbm_q"]) >= 0.843032 - 0.01, got["sbm_q"]
    assert got["star"] == [[0] * 41, [40, 0]]
