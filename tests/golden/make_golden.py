"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs the unmodified reference library (oracle/_ref/libnulpa_ref.so, built by
`make -C oracle` from /root/reference/proj/src) on small inputs and records its
outputs. Re-run here (where /root/reference exists):

    python tests/golden/make_golden.py

The GPU box never needs /root/reference: it reads the committed .npz files.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle as O  # noqa: E402

OUT = Path(__file__).resolve().parent

SEQ, SYNC = 1, 2


def edges_graph(edges, n=None):
    u = np.array([e[0] for e in edges], np.uint32)
    v = np.array([e[1] for e in edges], np.uint32)
    w = np.array([e[2] if len(e) > 2 else 1.0 for e in edges], np.float64)
    return O.RefGraph.from_edges(u, v, w, -1 if n is None else n)


def kat_graphs():
    cliques = []
    for s in (0, 5):
        for a in range(s, s + 5):
            for b in range(a + 1, s + 5):
                cliques.append((a, b))
    cliques.append((4, 5))
    return {
        "star3": O.RefGraph.star(3),
        "star40": O.RefGraph.star(40),
        "single_edge": edges_graph([(0, 1)]),
        "two_triangles": edges_graph([(0, 1), (1, 2), (0, 2), (3, 4), (4, 5), (3, 5)]),
        "k22": edges_graph([(0, 2), (0, 3), (1, 2), (1, 3)]),
        "bridged_cliques": edges_graph(cliques),
        "edgeless4": O.RefGraph.from_edges(np.zeros(0, np.uint32), np.zeros(0, np.uint32),
                                           None, 4),
        "ring_of_cliques": O.RefGraph.ring_of_cliques(6, 5),
    }


def random_graph(rng, n, p, weighted, loops):
    u, v, w = [], [], []
    for i in range(n):
        for j in range(i if loops else i + 1, n):
            if rng.random() < p:
                u.append(i)
                v.append(j)
                w.append(0.25 * (1 + rng.integers(0, 8)) if weighted else 1.0)
    return O.RefGraph.from_edges(np.array(u, np.uint32), np.array(v, np.uint32),
                                 np.array(w, np.float64), n)


CONFIGS = [dict(exec_mode=m, pl_period=pl, cc_period=cc, prune=pr)
           for m in (SEQ, SYNC) for pl in (0, 1, 4) for cc in (0, 1) for pr in (True, False)]


def record(name, g, rng, index, extra=None):
    off, tgt, w = g.arrays()
    data = {"offsets": off, "targets": tgt, "weights": w}
    runs = []
    for k, cfg in enumerate(CONFIGS):
        labels, st = O.ref_lpa(g, tolerance=1e-9 if cfg["exec_mode"] == SEQ else 0.05,
                               max_iterations=20, **cfg)
        data[f"run{k}_labels"] = labels
        runs.append({"config": cfg, "tolerance": 1e-9 if cfg["exec_mode"] == SEQ else 0.05,
                     **{kk: st[kk] for kk in ("iterations", "converged", "pl_iterations",
                                              "cc_reverts", "delta_n")}})
    steps = []
    if g.n > 0:
        for k in range(3):
            lab = rng.integers(0, g.n, g.n).astype(np.uint32) if k else np.arange(g.n, dtype=np.uint32)
            for pl in (0, 1):
                out, ch = O.ref_sync_step(g, lab, pl)
                data[f"step{k}_{pl}_in"] = lab
                data[f"step{k}_{pl}_out"] = out
                steps.append({"input": k, "pick_less": pl, "changed": ch})
    mods = []
    if g.m2 > 0:
        for k in range(2):
            lab = rng.integers(0, g.n, g.n).astype(np.uint32) if k else np.arange(g.n, dtype=np.uint32)
            data[f"mod{k}_labels"] = lab
            mods.append(O.ref_modularity(g, lab))
    # cross_check on a random (labels, prev, flags) triple
    cc = None
    if g.n > 1:
        prev = np.arange(g.n, dtype=np.uint32)
        lab = prev.copy()
        for i in range(g.n):
            nb = tgt[off[i]:off[i + 1]]
            if nb.size and rng.random() < 0.6:
                lab[i] = nb[rng.integers(0, nb.size)]
        flags = np.ones(g.n, np.uint8)
        data["cc_labels_in"] = lab.copy()
        data["cc_prev"] = prev
        rev = O.ref_cross_check(g, lab, prev, flags)
        data["cc_labels_out"] = lab
        data["cc_flags_out"] = flags
        cc = rev
    low, high = O.ref_partition(g, 3)
    data["part3_low"] = low
    data["part3_high"] = high
    np.savez_compressed(OUT / f"{name}.npz", **data)
    index[name] = {"n": g.n, "m2": g.m2, "total_2m": float(O.ref().ref_graph_total_2m(g.h)),
                   "runs": runs, "steps": steps, "modularity": mods, "cc_reverts": cc,
                   **(extra or {})}


def main():
    rng = np.random.default_rng(20241118)
    index = {}
    for name, g in kat_graphs().items():
        record(f"kat_{name}", g, rng, index)
    for k in range(12):
        n = int(rng.integers(8, 60))
        p = 0.08 if k % 2 == 0 else 0.25
        g = random_graph(rng, n, p, weighted=(k % 3 == 0), loops=(k % 4 == 3))
        record(f"random{k:02d}", g, rng, index, {"weighted": k % 3 == 0, "loops": k % 4 == 3})
    # The acceptance suite's parity graph (acceptance.cpp:63-68), seed 101.
    pin, pout = 0.15, (20.0 - 0.15 * 99.0) / 9900.0
    g = O.RefGraph.planted(10000, 100, pin, pout, 101)
    record("sbm10k_seed101", g, rng, index, {"planted": [10000, 100, pin, pout, 101]})
    # Probe-placement KATs on the reference hashtable (test_hashtable.cpp:71-107) as dumps.
    ht = []
    for strategy in range(4):
        for keys in ([0, 7, 14], [3, 10]):
            sk, sv, f = O.ref_ht_seq(7, 15, strategy, keys, [1.0] * len(keys))
            ht.append({"strategy": strategy, "keys": keys, "slots": sk.tolist(), "fail": f})
    index["_hashtable_placement"] = ht
    (OUT / "index.json").write_text(json.dumps(index, indent=1, sort_keys=True))
    total = sum(p.stat().st_size for p in OUT.glob("*.npz"))
    print(f"wrote {len(index)} fixtures, {total / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
