"""The position-order residency (layout.cu): results must not depend on the layout.

Under NULPA_LAYOUT_DEGREE_BUCKETS (the default) the resident rows are stored grouped by
degree bucket; label values stay vertex ids and every label array crossing the ABI is in
vertex order. These tests pin that: the downloaded CSR equals the identity-layout one, the
bit-exact gates give the same answers under both layouts, and the position/vertex
conversions invert each other.
"""
import numpy as np
import pytest

import oracle as O
from paper_2411_11468_b200 import _capi
from paper_2411_11468_b200 import labelprop as lp

pytestmark = pytest.mark.gpu


@pytest.fixture
def identity_layout():
    lp.set_default_layout(_capi.NULPA_LAYOUT_IDENTITY)
    yield
    lp.set_default_layout(_capi.NULPA_LAYOUT_DEGREE_BUCKETS)


def _gen(kind):
    if kind == "rmat":
        return lp.DeviceGraph.rmat(13, 16, 11)
    if kind == "web":
        return lp.DeviceGraph.web(20000, 160000, 2.1, 4, 5000, 3)
    return lp.DeviceGraph.grid(97, 41)


@pytest.mark.parametrize("kind", ["rmat", "web", "grid"])
def test_download_is_layout_independent(kind):
    dg = _gen(kind)
    assert dg.layout == _capi.NULPA_LAYOUT_DEGREE_BUCKETS
    a = dg.download()
    lp.set_default_layout(_capi.NULPA_LAYOUT_IDENTITY)
    try:
        di = _gen(kind)
        assert di.layout == _capi.NULPA_LAYOUT_IDENTITY
        b = di.download()
    finally:
        lp.set_default_layout(_capi.NULPA_LAYOUT_DEGREE_BUCKETS)
    assert np.array_equal(a.offsets, b.offsets) and np.array_equal(a.targets, b.targets)


def test_position_order_is_degree_bucketed():
    import torch
    dg = _gen("rmat")
    c = dg.device_csr()
    off = torch.empty(dg.n + 1, dtype=torch.int64, device="cuda:0")
    import cuda.bindings.runtime as rt
    err, = rt.cudaMemcpy(off.data_ptr(), c.offsets, (dg.n + 1) * 8,
                         rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice)
    assert err == rt.cudaError_t.cudaSuccess
    deg = (off[1:] - off[:-1]).cpu().numpy()
    bucket = np.where(deg == 0, -1, np.ceil(np.log2(np.maximum(deg, 1))).astype(int))
    assert (np.diff(bucket) <= 0).all()  # largest bucket first, isolated last
    # positions <-> vertices round trip, and vertex order is the input numbering
    vid = torch.arange(dg.n, dtype=torch.int32, device="cuda:0")
    pos = torch.empty_like(vid)
    back = torch.empty_like(vid)
    dg.labels_to_position_order(vid.data_ptr(), pos.data_ptr())
    dg.labels_to_vertex_order(pos.data_ptr(), back.data_ptr())
    assert torch.equal(back, vid)
    perm = pos.cpu().numpy()
    assert np.array_equal(np.sort(perm), np.arange(dg.n))
    g = dg.download()
    assert np.array_equal(np.diff(g.offsets.astype(np.int64))[perm], deg)


@pytest.mark.parametrize("kind", ["rmat", "web", "grid"])
def test_gates_identical_under_both_layouts(kind, identity_layout):
    di = _gen(kind)
    g = di.download()
    lp.set_default_layout(_capi.NULPA_LAYOUT_DEGREE_BUCKETS)
    pg = O.PortGraph(g.offsets, g.targets, None)
    rng = np.random.default_rng(5)
    lab = rng.integers(0, g.order(), g.order()).astype(np.uint32)
    for pl in (0, 1):
        want, wc = O.port_sync_step(pg, lab, pl)
        for layout in (_capi.NULPA_LAYOUT_IDENTITY, _capi.NULPA_LAYOUT_DEGREE_BUCKETS):
            lp.set_default_layout(layout)
            got, gc = lp.sync_step(g, lab, pl)
            assert gc == wc and np.array_equal(got, want), (kind, layout, pl)
    want, ws = O.port_lpa(pg, exec_mode=2, pl_period=4, cc_period=2)
    for layout in (_capi.NULPA_LAYOUT_IDENTITY, _capi.NULPA_LAYOUT_DEGREE_BUCKETS):
        lp.set_default_layout(layout)
        r = lp.lpa(g, lp.LpaConfig(exec=lp.ExecMode.Synchronous, pl_period=4, cc_period=2))
        assert np.array_equal(r.labels, want) and r.stats.delta_n_per_iter == ws["delta_n"]
        assert r.stats.cc_reverts == ws["cc_reverts"]


def test_async_labels_are_vertex_ids_in_vertex_order():
    dg = _gen("rmat")
    g = dg.download()
    r = dg.lpa(lp.LpaConfig())
    lab = r.labels
    assert lab.max() < g.order()
    # every vertex's label is the id of a vertex in its closed neighbourhood's label set:
    # at least, isolated vertices keep their own id (lpa.cpp:250-253)
    deg = np.diff(g.offsets.astype(np.int64))
    iso = np.flatnonzero(deg == 0)
    assert np.array_equal(lab[iso], iso.astype(np.uint32))
    q = lp.modularity(g, lab)
    assert abs(q - O.port_modularity(O.PortGraph(g.offsets, g.targets, None), lab)) < 1e-9


@pytest.mark.parametrize("chunk", ["1000", "7", "100000000"])
def test_pipelined_upload_matches_device_build(chunk, monkeypatch):
    """Host CSR upload streams the targets in row chunks and scatters each chunk into
    position order while the next is in flight; tiny chunks (and rows longer than a
    chunk) must give the same resident graph and the same results."""
    monkeypatch.setenv("NULPA_UPLOAD_CHUNK", chunk)
    dg = lp.DeviceGraph.web(20000, 160000, 2.1, 4, 5000, 3)
    g = dg.download()
    up = lp.DeviceGraph.upload(g)
    assert up.layout == _capi.NULPA_LAYOUT_DEGREE_BUCKETS
    assert up.max_degree == dg.max_degree
    h = up.download()
    assert np.array_equal(h.offsets, g.offsets) and np.array_equal(h.targets, g.targets)
    a = up.lpa(lp.LpaConfig(exec=lp.ExecMode.Synchronous))
    b = dg.lpa(lp.LpaConfig(exec=lp.ExecMode.Synchronous))
    assert np.array_equal(a.labels, b.labels)


def test_pipelined_upload_rejects_bad_targets():
    g = lp.CsrGraph(np.array([0, 2, 3, 4], np.uint64), np.array([1, 2, 0, 7], np.uint32))
    with pytest.raises(lp.ValidationError, match="out of range"):
        lp.DeviceGraph.upload(g)


@pytest.mark.parametrize("name", ["random00", "random03", "random06", "kat_star40"])
def test_pipelined_upload_golden_weighted(name, golden_index, monkeypatch):
    """Weighted (and unit) golden graphs through the chunked upload, 5-entry chunks:
    the reference's own Synchronous trajectories and modularity, bit for bit."""
    from conftest import load_golden
    monkeypatch.setenv("NULPA_UPLOAD_CHUNK", "5")
    meta = golden_index[name]
    d = load_golden(name)
    g = lp.CsrGraph(d["offsets"], d["targets"], d["weights"])
    for k, run in enumerate(meta["runs"]):
        c = run["config"]
        if c["exec_mode"] != 2:
            continue
        r = lp.lpa(g, lp.LpaConfig(exec=lp.ExecMode.Synchronous, pl_period=c["pl_period"],
                                   cc_period=c["cc_period"], prune=c["prune"],
                                   tolerance=run["tolerance"]))
        assert np.array_equal(r.labels, d[f"run{k}_labels"]), (name, c)
        assert r.stats.delta_n_per_iter == run["delta_n"]
    for k, q in enumerate(meta["modularity"]):
        assert abs(lp.modularity(g, d[f"mod{k}_labels"]) - q) < 1e-12


def test_pipelined_upload_many_long_row_spans(monkeypatch):
    """More long-row spans than warps in the scatter grid (each warp walks several
    4096-entry spans): R-MAT scale 20 in one chunk and in small chunks."""
    dg = lp.DeviceGraph.rmat(20, 16, 1)
    g = dg.download()
    dg.free()
    for chunk in (None, "300000"):
        if chunk:
            monkeypatch.setenv("NULPA_UPLOAD_CHUNK", chunk)
        up = lp.DeviceGraph.upload(lp.CsrGraph(g.offsets, g.targets, None))
        h = up.download()
        assert np.array_equal(h.offsets, g.offsets) and np.array_equal(h.targets, g.targets)
        up.free()
