"""Pin the C restatement (oracle/oracle.c) before trusting it (CPU only).

1. Known-answer tests copied as literal expectations from the reference's own
   suites (proj/tests/test_lpa.cpp, test_hashtable.cpp, test_quality.cpp).
2. Golden vectors produced by the reference itself (tests/golden/, made by
   tests/golden/make_golden.py from oracle/_ref).
3. When oracle/_ref is built here, direct port-vs-reference runs on fresh inputs.
"""
import numpy as np
import pytest

import oracle as O
from conftest import golden_names, load_golden

STRATS = range(4)


def pg_of(data):
    return O.PortGraph(data["offsets"], data["targets"], data["weights"])


# ---- KATs (literal values from the reference test suites) ------------------------


def test_geometry_kats():
    # test_hashtable.cpp:30-52: degree 7 -> (7, 15), 1 -> (1, 3), 8 -> (15, 31)
    assert O.port_geometry(7) == (7, 15)
    assert O.port_geometry(1) == (1, 3)
    assert O.port_geometry(8) == (15, 31)
    assert O.port_geometry(0) is None
    for d in range(1, 201):
        p1, _ = O.port_geometry(d)
        assert d <= p1 <= 2 * d - 1


@pytest.mark.parametrize("strategy,slot7,slot14", [(0, 1, 2), (1, 1, 3), (2, 1, 2), (3, 1, 3)])
def test_probe_placement_kat(strategy, slot7, slot14):
    # test_hashtable.cpp:71-94: keys 0, 7, 14 in a 7-slot region.
    sk, _, f = O.port_ht_seq(7, 15, strategy, [0, 7, 14], [1.0, 1.0, 1.0])
    assert f == 0
    slots = {int(k): s for s, k in enumerate(sk) if k != 0xFFFFFFFF}
    assert slots == {0: 0, 7: slot7, 14: slot14}


def test_quadratic_double_first_advance_kat():
    # test_hashtable.cpp:96-107: key 10 lands after key 3 at slot 4.
    sk, _, _ = O.port_ht_seq(7, 15, 3, [3, 10], [1.0, 1.0])
    assert sk[3] == 3 and sk[4] == 10


def test_overflow_reports_failure():
    # test_hashtable.cpp:218-234: a 4th distinct key in p1=3 fails.
    for s in STRATS:
        sk, sv, f = O.port_ht_seq(3, 7, s, [1, 2, 3, 4], [1.0] * 4)
        assert f == 1
        assert sorted(int(k) for k in sk) == [1, 2, 3]


def test_full_load_and_residue_pileup():
    # test_hashtable.cpp:170-216
    rng = np.random.default_rng(2024)
    for p1 in (1, 3, 7, 15, 31, 63, 127):
        for s in STRATS:
            keys = rng.choice(0xFFFFFFFE, size=p1, replace=False).astype(np.uint32)
            _, _, f = O.port_ht_seq(p1, 2 * (p1 + 1) - 1, s, np.concatenate([keys, keys]),
                                    np.ones(2 * p1, np.float32))
            assert f == 0
    for s in STRATS:
        keys = (np.arange(63, dtype=np.uint64) * 63).astype(np.uint32)
        _, _, f = O.port_ht_seq(63, 127, s, keys, np.ones(63, np.float32))
        assert f == 0


def _edges(edges, n=None):
    n = n if n is not None else 1 + max(max(a, b) for a, b in edges)
    adj = [[] for _ in range(n)]
    for a, b in edges:
        adj[a].append(b)
        if a != b:
            adj[b].append(a)
    off = np.zeros(n + 1, np.uint64)
    tgt = []
    for i in range(n):
        row = sorted(set(adj[i]))
        tgt.extend(row)
        off[i + 1] = off[i] + len(row)
    return O.PortGraph(off, np.array(tgt, np.uint32))


def test_lpa_kats():
    star3 = _edges([(0, 1), (0, 2), (0, 3)])
    lab, st = O.port_lpa(star3, exec_mode=1, pl_period=0)
    assert lab.tolist() == [1, 1, 1, 1] and st["delta_n"] == [3, 0] and st["converged"]
    lab, st = O.port_lpa(star3, exec_mode=1, pl_period=4)
    assert lab.tolist() == [0, 0, 0, 0] and st["pl_iterations"] == 1
    tri = _edges([(0, 1), (1, 2), (0, 2), (3, 4), (4, 5), (3, 5)])
    assert O.port_lpa(tri, exec_mode=1, pl_period=0)[0].tolist() == [1, 1, 1, 4, 4, 4]
    assert O.port_lpa(tri, exec_mode=1, pl_period=4)[0].tolist() == [0, 0, 0, 3, 3, 3]
    k22 = _edges([(0, 2), (0, 3), (1, 2), (1, 3)])
    lab, st = O.port_lpa(k22, exec_mode=2, pl_period=0)
    assert not st["converged"] and st["iterations"] == 20 and st["delta_n"] == [4] * 20
    assert lab.tolist() == [0, 0, 2, 2]
    lab, st = O.port_lpa(k22, exec_mode=2, pl_period=0, cc_period=1)
    assert st["converged"] and st["delta_n"] == [2, 1, 0] and st["cc_reverts"] == 2
    assert lab.tolist() == [2, 2, 2, 2]
    edge = _edges([(0, 1)])
    lab, st = O.port_lpa(edge, exec_mode=2, pl_period=0, cc_period=1)
    assert st["delta_n"] == [1, 0] and st["cc_reverts"] == 1 and lab.tolist() == [1, 1]
    lab, st = O.port_lpa(k22, exec_mode=2, pl_period=1)
    assert lab.tolist() == [0, 0, 0, 0] and st["delta_n"][:2] == [2, 1]


def test_modularity_kats():
    # test_quality.cpp:37-49
    e = []
    for s in (0, 5):
        for a in range(s, s + 5):
            for b in range(a + 1, s + 5):
                e.append((a, b))
    e.append((4, 5))
    g = _edges(e)
    assert abs(O.port_modularity(g, [0] * 5 + [5] * 5) - 19 / 42) < 1e-12
    assert O.port_modularity(_edges([(0, 1)]), [0, 1]) == -0.5


def test_cross_check_kat():
    # test_lpa.cpp:88-108
    g = _edges([(0, 1)])
    lab = np.array([1, 0], np.uint32)
    flags = np.array([1, 1], np.uint8)
    assert O.port_cross_check(g, lab, [0, 1], flags) == 1
    assert lab.tolist() == [1, 1] and flags.tolist() == [0, 0]


# ---- golden vectors from the reference -------------------------------------------


@pytest.mark.parametrize("name", golden_names())
def test_port_matches_golden(name, golden_index):
    meta = golden_index[name]
    d = load_golden(name)
    g = pg_of(d)
    for k, run in enumerate(meta["runs"]):
        cfg = run["config"]
        lab, st = O.port_lpa(g, exec_mode=cfg["exec_mode"], pl_period=cfg["pl_period"],
                             cc_period=cfg["cc_period"], prune=cfg["prune"],
                             tolerance=run["tolerance"], max_iterations=20)
        assert np.array_equal(lab, d[f"run{k}_labels"]), (name, cfg)
        for key in ("iterations", "converged", "pl_iterations", "cc_reverts", "delta_n"):
            assert st[key] == run[key], (name, cfg, key)
    for st in meta["steps"]:
        k, pl = st["input"], st["pick_less"]
        out, ch = O.port_sync_step(g, d[f"step{k}_{pl}_in"], pl)
        assert ch == st["changed"] and np.array_equal(out, d[f"step{k}_{pl}_out"])
    for k, q in enumerate(meta["modularity"]):
        assert abs(O.port_modularity(g, d[f"mod{k}_labels"]) - q) < 1e-12
    if meta["cc_reverts"] is not None:
        lab = d["cc_labels_in"].copy()
        flags = np.ones(g.n, np.uint8)
        assert O.port_cross_check(g, lab, d["cc_prev"], flags) == meta["cc_reverts"]
        assert np.array_equal(lab, d["cc_labels_out"])
        assert np.array_equal(flags, d["cc_flags_out"])
    low, high = O.port_partition(g, 3)
    assert np.array_equal(low, d["part3_low"]) and np.array_equal(high, d["part3_high"])


def test_golden_hashtable_placement(golden_index):
    for case in golden_index["_hashtable_placement"]:
        sk, _, f = O.port_ht_seq(7, 15, case["strategy"], case["keys"],
                                 [1.0] * len(case["keys"]))
        assert f == case["fail"] and sk.tolist() == case["slots"]


# ---- direct port vs reference (only where oracle/_ref was built) ----------------------


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_port_vs_reference_sbm_sync_trajectory():
    # SURVEY §8c gate 2 known value: SBM seed 1 -> 10 iterations, Q = 0.843032.
    g = O.RefGraph.planted(100000, 100, 14 / 999, 2 / 99000, 1)
    off, tgt, w = g.arrays()
    pg = O.PortGraph(off, tgt, w)
    lr, sr = O.ref_lpa(g, exec_mode=2)
    lp, sp = O.port_lpa(pg, exec_mode=2)
    assert np.array_equal(lr, lp)
    assert sr["delta_n"] == sp["delta_n"] == [96812, 96437, 97578, 94668, 56403, 43148, 21383,
                                              10307, 3096, 2503]
    assert abs(O.port_modularity(pg, lp) - 0.843032184933054) < 1e-12
