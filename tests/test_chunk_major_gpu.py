"""The chunk-major low range (layout.cu chunk_major): on graphs whose rows of degree <= 8
carry most of the entries, those rows are stored transposed for the chunk walk of the
thread tier (entry k*L + r of the bucket order at column r, row k), so the walk's loads
coalesce. Only positions move: the layout must be exactly that permutation, label arrays
still cross the ABI in vertex order, the bit-exact gates must not see it, and the
ParallelAsync chunk walk (the reference's per-worker slices, lpa.cpp:139-165) must still
converge on a lattice.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from conftest import ROOT

import oracle as O
from paper_2411_11468_b200 import _capi
from paper_2411_11468_b200 import labelprop as lp

pytestmark = pytest.mark.gpu


def _positions(dg):
    """perm as an array: perm[p] = vertex id stored at position p."""
    vid = torch.arange(dg.n, dtype=torch.int32, device="cuda:0")
    pos = torch.empty_like(vid)
    dg.labels_to_position_order(vid.data_ptr(), pos.data_ptr())
    return pos.cpu().numpy().astype(np.int64)


def _expected_perm(g, sms):
    """Bucket order (ceil(log2 deg) descending, isolated last, ascending id inside a
    bucket), then the degree-1..8 range transposed into L = max(ceil(M / (sms * 1024)), 32)
    columns."""
    deg = np.diff(g.offsets.astype(np.int64))
    key = np.where(deg == 0, 40, 33 - np.where(deg <= 1, 0, np.ceil(np.log2(np.maximum(deg, 1)))))
    perm = np.argsort(key, kind="stable")
    a = int((deg > 8).sum())
    M = int(((deg >= 1) & (deg <= 8)).sum())
    L = max(-(-M // (sms * 1024)), 32)
    q, rem = divmod(M, L)
    out = perm.copy()
    for r in range(L):
        rows = q + (1 if r < rem else 0)
        start = r * q + min(r, rem)
        k = np.arange(rows)
        out[a + start + k] = perm[a + k * L + r]
    return out, L


@pytest.mark.parametrize("shape", [(512, 512), (1000, 333)])
def test_chunk_major_layout_is_the_transposed_bucket_order(shape):
    dg = lp.DeviceGraph.grid(*shape)
    g = dg.download()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    want, L = _expected_perm(g, sms)
    assert L >= 2
    assert np.array_equal(_positions(dg), want)


def test_chunk_major_gates_match_identity_layout():
    dg = lp.DeviceGraph.grid(600, 400)
    g = dg.download()
    pg = O.PortGraph(g.offsets, g.targets, None)
    lab = np.random.default_rng(3).integers(0, g.order(), g.order()).astype(np.uint32)
    for pl in (False, True):
        got, gc = lp.sync_step(g, lab, pick_less=pl)
        want, wc = O.port_sync_step(pg, lab, 1 if pl else 0)
        assert gc == wc and np.array_equal(got, want)
    r = dg.lpa(lp.LpaConfig(exec=lp.ExecMode.Synchronous))
    lp.set_default_layout(_capi.NULPA_LAYOUT_IDENTITY)
    try:
        di = lp.DeviceGraph.grid(600, 400)
        ri = di.lpa(lp.LpaConfig(exec=lp.ExecMode.Synchronous))
    finally:
        lp.set_default_layout(_capi.NULPA_LAYOUT_DEGREE_BUCKETS)
    assert np.array_equal(r.labels, ri.labels)
    assert r.stats.delta_n_per_iter == ri.stats.delta_n_per_iter


CHILD = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
from paper_2411_11468_b200 import labelprop as lp
dg = lp.DeviceGraph.grid(2048, 2048)
g = dg.download()
out = []
for _ in range(2):
    r = dg.lpa(lp.LpaConfig())
    out.append([bool(r.stats.converged), r.stats.iterations, lp.modularity(g, r.labels)])
print(json.dumps(out))
"""


def _lattice_runs(**env):
    e = dict(os.environ)
    e.update({k: str(v) for k, v in env.items()})
    p = subprocess.run([sys.executable, "-c", CHILD, str(ROOT)], env=e, capture_output=True,
                       text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


def test_chunk_major_async_lattice_converges():
    """The chunk walk over the chunk-major range (grouped k_chunk_walk and the one-row
    k_thread walk) converges like the same walk over the bucket-order layout."""
    base = _lattice_runs(NULPA_CHUNK_MAJOR=0)
    q0 = np.mean([q for _, _, q in base])
    assert all(c and it < 20 for c, it, _ in base), base
    for env in ({}, {"NULPA_CHUNK_ROWS": 1}, {"NULPA_CHUNK_ROWS": 4}, {"NULPA_CHUNK_ROWS": 8},
                {"NULPA_CHUNK_ROWS": 14}):
        got = _lattice_runs(**env)
        assert all(c and it < 20 for c, it, _ in got), (env, got)
        assert abs(np.mean([q for _, _, q in got]) - q0) <= 0.01, (env, got, base)
