"""community_stats / |Γ| and membership I/O.

community_stats (quality.cpp:56-78) runs on the device and is checked against a numpy
restatement on golden and generated graphs; delta_modularity (quality.cpp:51-54) against
the reference's own ΔQ-vs-Q-difference property (test_quality.cpp:83-119); membership I/O
(io.cpp) by round trip and the reference's error messages.
"""
import numpy as np
import pytest

from conftest import load_golden
from paper_2411_11468_b200 import labelprop as lp


def _np_stats(g, lab):
    off = g.offsets.astype(np.int64)
    src = np.repeat(np.arange(g.order()), np.diff(off))
    w = g.weights.astype(np.float64)
    comms, sizes = np.unique(lab, return_counts=True)
    big = np.zeros(g.order())
    np.add.at(big, lab[src], w)
    sig = np.zeros(g.order())
    intra = lab[src] == lab[g.targets]
    np.add.at(sig, lab[src][intra], w[intra])
    hist_s, hist_c = np.unique(sizes, return_counts=True)
    return (comms.size, dict(zip(hist_s.tolist(), hist_c.tolist())),
            {int(c): sig[c] for c in comms}, {int(c): big[c] for c in comms})


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["random00", "random03", "sbm10k_seed101", "kat_star40"])
def test_community_stats_matches_restatement(name):
    d = load_golden(name)
    g = lp.CsrGraph(d["offsets"], d["targets"], d["weights"])
    rng = np.random.default_rng(1)
    for lab in (np.arange(g.order(), dtype=np.uint32),
                (rng.integers(0, 7, g.order()) * 3).astype(np.uint32),
                lp.lpa(g).labels):
        st = lp.community_stats(g, lab)
        cnt, hist, sig, big = _np_stats(g, lab.astype(np.int64))
        assert st.count == cnt == lp.community_count(g, lab)
        assert st.size_histogram == hist
        assert st.sigma.keys() == sig.keys() and st.big_sigma.keys() == big.keys()
        for c in sig:
            assert abs(st.sigma[c] - sig[c]) <= 1e-9 * max(1.0, abs(sig[c]))
            assert abs(st.big_sigma[c] - big[c]) <= 1e-9 * max(1.0, abs(big[c]))


@pytest.mark.gpu
def test_community_stats_large_generated():
    dg = lp.DeviceGraph.rmat(16, 16, 3)
    g = dg.download()
    lab = dg.lpa(lp.LpaConfig()).labels
    st = lp.community_stats(g, lab)
    cnt, hist, sig, big = _np_stats(g, lab.astype(np.int64))
    assert st.count == cnt and st.size_histogram == hist
    assert max(abs(st.sigma[c] - sig[c]) for c in sig) < 1e-6


@pytest.mark.gpu
def test_delta_modularity_matches_q_difference():
    # test_quality.cpp:83-119: moving one vertex changes Q by exactly delta_modularity
    d = load_golden("kat_bridged_cliques")
    g = lp.CsrGraph(d["offsets"], d["targets"], d["weights"])
    n = g.order()
    lab = np.array([0] * (n // 2) + [n // 2] * (n - n // 2), np.uint32)
    m = g.total_weight_2m() / 2
    q0 = lp.modularity(g, lab)
    i, c, dd = 0, n // 2, 0
    nb, wt = g.neighbors(i), g.weights[g.offsets[i]:g.offsets[i + 1]].astype(np.float64)
    ki = wt.sum()
    to_c = wt[(lab[nb] == c) & (nb != i)].sum()
    to_d = wt[(lab[nb] == dd) & (nb != i)].sum()
    st = lp.community_stats(g, lab)
    dq = lp.delta_modularity(m, ki, to_c, to_d, st.big_sigma[c], st.big_sigma[dd])
    moved = lab.copy()
    moved[i] = c
    assert abs(lp.modularity(g, moved) - q0 - dq) < 1e-12


@pytest.mark.gpu
def test_membership_round_trip(tmp_path):
    lab = np.array([3, 3, 0, 1], np.uint32)
    p = tmp_path / "m.tsv"
    lp.write_membership(p, lab)  # formatted on the device
    assert p.read_text() == "0\t3\n1\t3\n2\t0\n3\t1\n"
    assert np.array_equal(lp.read_membership(p, 4), lab)


def test_membership_read_and_errors(tmp_path):
    lab = np.array([3, 3, 0, 1], np.uint32)
    p = tmp_path / "m.tsv"
    p.write_text("0\t3\n1 3\n# c\n  2\t0  \n3\t1")
    assert np.array_equal(lp.read_membership(p, 4), lab)
    cases = {
        "1\t2\t3\n": (lp.FormatError, "trailing content after label"),
        "x\t1\n": (lp.FormatError, "expected 'vertex<TAB>label'"),
        "5\t0\n": (lp.ValidationError, "vertex 5 out of range for n=4"),
        "0\t9\n": (lp.ValidationError, "label 9 out of range for n=4"),
        "0\t1\n0\t1\n": (lp.ValidationError, "vertex 0 assigned twice"),
        "# c\n0 1\n1 1\n2 1\n": (lp.ValidationError, "no label for vertex 3"),
    }
    for text, (err, msg) in cases.items():
        q = tmp_path / "bad.tsv"
        q.write_text(text)
        with pytest.raises(err, match=msg):
            lp.read_membership(q, 4)
