"""The asynchronous label/flag protocol (reference lpa.cpp:44-60,
:143-147, :161-163).

The reference makes every label and flag access seq_cst so that "a stale read is always
re-examined": when a vertex keeps its processed flag at the end of a pass, no neighbour
label it read can have changed after it read it. Consequence (the pruning invariant):
after a non-Pick-Less ParallelAsync pass with wake-ups on, every non-isolated vertex
whose flag is still 1 makes NO move when its rule is recomputed from the end-of-pass
labels. The GPU keeps the invariant with relaxed device-scope label/flag accesses and a
fence.sc between each claim (or label change) and the loads that depend on it
(device.cuh, lpa_kernels.cuh). This test drives single passes through the session API
and recomputes every flagged vertex's rule with the bit-exact synchronous step (itself
gated against the C restatement in test_parity_gpu.py).
"""
import numpy as np
import pytest

import oracle as O
from paper_2411_11468_b200 import labelprop as lp

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _vertex_order_flags(dg, flags_pos):
    """Session flags are in position order; map them to vertex order."""
    n = dg.n
    iota = torch.arange(n, dtype=torch.int32, device=f"cuda:{dg.device}")
    pos_of = torch.empty_like(iota)
    dg.labels_to_vertex_order(iota.data_ptr(), pos_of.data_ptr())  # pos_of[v] = position of v
    return flags_pos[pos_of.long()]


def _check_invariant(dg, eng, deg_pos_nonzero, rng, passes=4):
    from paper_2411_11468_b200.dist import DeviceRangeEngine  # noqa: F401
    n = dg.n
    eng.init()
    # pass 0: Pick-Less (the schedule's first pass), then the post-PL flag reset
    eng.pass_(True, True)
    eng.flags.zero_()
    checked = 0
    for it in range(passes):
        info = eng.pass_(False, True)
        torch.cuda.synchronize()
        lab_v = eng.vertex_labels()
        flags_v = _vertex_order_flags(dg, eng.flags)
        out = torch.empty_like(lab_v)
        dg.sync_step_device(lab_v.data_ptr(), out.data_ptr(), False)
        flagged = (flags_v == 1) & deg_pos_nonzero
        moved = flagged & (out != lab_v)
        assert int(moved.sum()) == 0, (
            f"pass {it + 1}: {int(moved.sum())} flagged vertices would still move "
            f"(changed={info['changed']})")
        checked += int(flagged.sum())
        if info["changed"] == 0:
            break
    return checked


def _engine(dg):
    from paper_2411_11468_b200.dist import DeviceRangeEngine
    return DeviceRangeEngine(dg, lp.LpaConfig(), 0, dg.n)


def _nonisolated(dg):
    g = dg.download()
    deg = np.diff(g.offsets.astype(np.int64))
    return torch.from_numpy(deg > 0).to(f"cuda:{dg.device}"), g


@pytest.mark.parametrize("seed", range(20))
def test_pruning_invariant_rmat18(seed):
    dg = lp.DeviceGraph.rmat(18, 16, seed=100 + seed)
    nz, _ = _nonisolated(dg)
    eng = _engine(dg)
    try:
        assert _check_invariant(dg, eng, nz, np.random.default_rng(seed)) > 0
    finally:
        eng.free()


@pytest.mark.skipif(not O.ref_available(), reason="needs oracle/_ref (planted partition)")
@pytest.mark.parametrize("seed", range(1, 21))
def test_pruning_invariant_sbm100k(seed):
    off, tgt, _ = O.RefGraph.planted(100000, 100, 14 / 999, 2 / 99000, seed).arrays()
    dg = lp.DeviceGraph.upload(lp.CsrGraph(off, tgt, None))
    nz, _ = _nonisolated(dg)
    eng = _engine(dg)
    try:
        assert _check_invariant(dg, eng, nz, np.random.default_rng(seed)) > 0
    finally:
        eng.free()


@pytest.mark.parametrize("seed", range(20))
def test_pruning_invariant_grid(seed):
    # the lattice starts from a random labelling (seeded) so every seed is a new race
    dg = lp.DeviceGraph.grid(512, 512)
    nz, _ = _nonisolated(dg)
    eng = _engine(dg)
    try:
        eng.init()
        rng = np.random.default_rng(seed)
        lab = torch.from_numpy(rng.integers(0, dg.n, dg.n).astype(np.int32)).cuda()
        dg.labels_to_position_order(lab.data_ptr(), eng.labels.data_ptr())
        eng.flags.zero_()
        checked = 0
        for it in range(6):
            info = eng.pass_(False, True)
            torch.cuda.synchronize()
            lab_v = eng.vertex_labels()
            flags_v = _vertex_order_flags(dg, eng.flags)
            out = torch.empty_like(lab_v)
            dg.sync_step_device(lab_v.data_ptr(), out.data_ptr(), False)
            flagged = (flags_v == 1) & nz
            assert int((flagged & (out != lab_v)).sum()) == 0, f"pass {it}"
            checked += int(flagged.sum())
            if info["changed"] == 0:
                break
        assert checked > 0
    finally:
        eng.free()


def test_invariant_recompute_matches_port():
    # the recomputation itself: the device sync step on end-of-pass labels equals the C
    # restatement's (one R-MAT pass state)
    dg = lp.DeviceGraph.rmat(14, 16, seed=7)
    g = dg.download()
    eng = _engine(dg)
    try:
        eng.init()
        eng.pass_(True, True)
        eng.flags.zero_()
        eng.pass_(False, True)
        lab = eng.vertex_labels().cpu().numpy().view(np.uint32)
        want, _ = O.port_sync_step(O.PortGraph(g.offsets, g.targets, None), lab, 0)
        got, _ = lp.sync_step(g, lab, False)
        assert np.array_equal(got, want)
    finally:
        eng.free()
