"""Parity gates at the BASELINE.json configuration sizes, against the reference library
itself (oracle/_ref, the unmodified reference compiled from /root/reference/proj/src).

SURVEY §8c gate 1 (single synchronous step, bit-exact: labels and changed count) on
  * SBM-100K: planted_partition(100000, 100, 14/999, 2/99000, seed 1) (generators.cpp:45-88),
  * R-MAT scale 24, edgefactor 16 (m2 ~ 521M; the gate's largest size, "run gate 1 at R24
    and below"),
  * the 4096 x 4096 lattice (16.7M vertices),
  * a Chung-Lu power-law graph with hubs of degree > 1M (the web-like config's hub path),
with identity labels, seeded random labels and the reference's own mid-run labels, Pick-Less
on and off. The oracle is ref_sync_step: the reference's scan_candidate (lpa.hpp:92-111)
with a snapshot reader and sync_move's rule (lpa.cpp:87-88).

Gate 2 on SBM-100K: the full Synchronous trajectory against the reference's lpa() and the
survey's known values (10 iterations, dN = [96812, ..., 2503], Q = 0.843032).
"""
import numpy as np
import pytest

import oracle as O
from paper_2411_11468_b200 import labelprop as lp

pytestmark = [pytest.mark.gpu, pytest.mark.large,
              pytest.mark.skipif(not O.ref_available(), reason="needs oracle/_ref")]

SBM_DN = [96812, 96437, 97578, 94668, 56403, 43148, 21383, 10307, 3096, 2503]


def _gate(g_host, ref_graph, labels, what):
    for pl in (0, 1):
        want, wc = O.ref_sync_step(ref_graph, labels, pl)
        got, gc = lp.sync_step(g_host, labels, bool(pl))
        assert gc == wc, f"{what} pl={pl}: changed {gc} vs reference {wc}"
        bad = np.flatnonzero(got != want)
        assert bad.size == 0, f"{what} pl={pl}: {bad.size} labels differ, first at {bad[:5]}"


def _label_sets(n, rng, ref_graph, midrun_steps=2):
    sets = {"identity": np.arange(n, dtype=np.uint32),
            "random": rng.integers(0, n, n).astype(np.uint32),
            "clustered": (rng.integers(0, max(1, n // 1000), n) * 997 % n).astype(np.uint32)}
    # the reference's own synchronous steps from identity (PL first, as run_engine does)
    lab = sets["identity"]
    for k in range(midrun_steps):
        lab, _ = O.ref_sync_step(ref_graph, lab, 1 if k == 0 else 0)
    sets["ref_midrun"] = lab
    return sets


@pytest.fixture(scope="module")
def sbm():
    rg = O.RefGraph.planted(100000, 100, 14 / 999, 2 / 99000, 1)
    off, tgt, w = rg.arrays()
    return rg, lp.CsrGraph(off, tgt, None)


def test_sbm100k_sync_step_vs_reference(sbm):
    rg, g = sbm
    rng = np.random.default_rng(1)
    sets = _label_sets(g.order(), rng, rg, midrun_steps=0)
    # the reference's Synchronous run stopped after 2, 4 and 7 iterations
    for k in (2, 4, 7):
        sets[f"ref_sync_{k}"], _ = O.ref_lpa(rg, exec_mode=2, max_iterations=k)
    for name, lab in sets.items():
        _gate(g, rg, lab, f"sbm100k/{name}")


def test_sbm100k_sync_trajectory_vs_reference(sbm):
    rg, g = sbm
    want, ws = O.ref_lpa(rg, exec_mode=2)
    assert ws["delta_n"] == SBM_DN  # the survey's probe value (pins the oracle)
    r = lp.lpa(g, lp.LpaConfig(exec=lp.ExecMode.Synchronous))
    assert r.stats.delta_n_per_iter == SBM_DN
    assert r.stats.iterations == ws["iterations"] and r.stats.converged == ws["converged"]
    assert r.stats.pl_iterations == ws["pl_iterations"]
    assert np.array_equal(r.labels, want)
    q = lp.modularity(g, r.labels)
    assert abs(q - O.ref_modularity(rg, want)) < 1e-12
    assert abs(q - 0.843032) < 5e-7
    assert lp.community_stats(g, r.labels).count == 78


def test_rmat24_sync_step_vs_reference():
    dg = lp.DeviceGraph.rmat(24, 16, seed=1)
    g = dg.download()
    dg.free()
    assert g.directed_size() > 500_000_000
    rg = O.RefGraph.from_csr(g.offsets, g.targets, None)
    rng = np.random.default_rng(24)
    for name, lab in _label_sets(g.order(), rng, rg).items():
        _gate(g, rg, lab, f"rmat24/{name}")


def test_grid4096_sync_step_vs_reference():
    dg = lp.DeviceGraph.grid(4096, 4096)
    g = dg.download()
    dg.free()
    rg = O.RefGraph.from_csr(g.offsets, g.targets, None)
    rng = np.random.default_rng(4096)
    for name, lab in _label_sets(g.order(), rng, rg, midrun_steps=3).items():
        _gate(g, rg, lab, f"grid4096/{name}")


def test_web_hubs_over_1m_sync_step_vs_reference():
    # Chung-Lu power law with 3 hubs of expected degree 2.5M (distinct neighbours > 1M
    # after dedup): the hub tier's global tables
    dg = lp.DeviceGraph.web(16_000_000, 24_000_000, 2.1, 3, 2_500_000, seed=5)
    g = dg.download()
    dg.free()
    deg = np.diff(g.offsets.astype(np.int64))
    assert int((deg > 1_000_000).sum()) >= 2
    rg = O.RefGraph.from_csr(g.offsets, g.targets, None)
    rng = np.random.default_rng(5)
    for name, lab in _label_sets(g.order(), rng, rg).items():
        _gate(g, rg, lab, f"web/{name}")
