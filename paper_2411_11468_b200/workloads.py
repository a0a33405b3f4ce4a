"""The BASELINE.json input shapes, built on the device.

    rmat   Graph500 R-MAT, scale s, edgefactor 16 (A=.57 B=.19 C=.19 D=.05), seeded
           vertex permutation, symmetrised, deduplicated, unit weights (nulpa_gen_rmat)
    grid   rows x cols 4-neighbour lattice (nulpa_gen_grid); BASELINE: 4096 x 4096
    web    Chung-Lu power law, 50M vertices, ~1B undirected draws, gamma 2.1, hubs forced to
           degree 2M (nulpa_gen_web)
    sbm    planted partition (n vertices in k equal blocks, p_in / p_out), built from a host
           edge list by nulpa_graph_from_edges; BASELINE: n=100K, k=100, avg degree 16

Each workload also names the bounded CPU sample the reference's CPU path is timed on.
"""
from __future__ import annotations

import numpy as np

from . import labelprop as lp


def planted_partition_edges(n: int, k: int, p_in: float, p_out: float, seed: int):
    """Planted partition edge list (u < v), vectorised: Bernoulli(p_in) over every
    intra-block pair, Binomial-count uniform pairs across blocks (duplicates are dropped by
    the CSR build). Statistically the reference's planted_partition
    (generators.cpp:45-88); not the same random stream."""
    rng = np.random.default_rng(seed)
    base, rem = divmod(n, k)
    sizes = np.array([base + (1 if b < rem else 0) for b in range(k)])
    starts = np.concatenate([[0], np.cumsum(sizes)[:-1]])
    us, vs = [], []
    for b in range(k):
        sz, s0 = int(sizes[b]), int(starts[b])
        iu, ju = np.triu_indices(sz, 1)
        keep = rng.random(iu.size) < p_in
        us.append(iu[keep] + s0)
        vs.append(ju[keep] + s0)
    cross_pairs = (n * n - int((sizes * sizes).sum())) // 2
    m_out = rng.binomial(cross_pairs, p_out)
    block_of = np.repeat(np.arange(k), sizes)
    u = rng.integers(0, n, 2 * m_out + 16)
    v = rng.integers(0, n, 2 * m_out + 16)
    ok = block_of[u] != block_of[v]
    u, v = u[ok][:m_out], v[ok][:m_out]
    us.append(np.minimum(u, v))
    vs.append(np.maximum(u, v))
    return (np.concatenate(us).astype(np.uint32), np.concatenate(vs).astype(np.uint32),
            block_of.astype(np.uint32))


def build(name: str, scale: int = 27, seed: int = 1, device: int = 0):
    """The headline-sized workload `name` as a DeviceGraph, plus a description dict."""
    if name == "rmat":
        dg = lp.DeviceGraph.rmat(scale, 16, seed, device)
        return dg, {"workload": f"rmat{scale}-ef16", "generator": "nulpa_gen_rmat"}
    if name == "grid":
        dg = lp.DeviceGraph.grid(4096, 4096, device)
        return dg, {"workload": "grid-4096x4096", "generator": "nulpa_gen_grid"}
    if name == "web":
        dg = lp.DeviceGraph.web(50_000_000, 1_000_000_000, 2.1, 16, 2_000_000, seed, device)
        return dg, {"workload": "web-chunglu-50M-1B", "generator": "nulpa_gen_web",
                    "hubs": "16 vertices forced to degree ~2M"}
    if name == "sbm":
        u, v, _ = planted_partition_edges(100_000, 100, 14 / 999, 2 / 99000, seed)
        dg = lp.DeviceGraph.from_edges(u, v, 100_000, device)
        return dg, {"workload": "sbm-100K-k100-deg16", "generator": "planted_partition_edges"}
    raise ValueError(f"unknown workload {name}")


def cpu_sample(name: str, ref_scale: int = 22, seed: int = 1, device: int = 0):
    """A bounded sample of the same workload for the reference CPU path (host CSR)."""
    if name == "rmat":
        dg = lp.DeviceGraph.rmat(ref_scale, 16, seed, device)
        desc = f"R-MAT scale-{ref_scale} ef16"
    elif name == "grid":
        dg = lp.DeviceGraph.grid(1024, 1024, device)
        desc = "grid 1024x1024"
    elif name == "web":
        dg = lp.DeviceGraph.web(2_000_000, 40_000_000, 2.1, 4, 100_000, seed, device)
        desc = "web Chung-Lu 2M vertices / 40M draws"
    else:
        dg, _ = build("sbm", seed=seed, device=device)
        desc = "the full SBM"
    g = dg.download()
    dg.free()
    return g, desc


def export_csr(name: str, scale: int, seed: int, out_dir: str, device: int = 0) -> dict:
    """Build the workload on the device and write its host CSR as raw arrays
    (`offsets.u64`, `targets.u32`, `meta.json`) into out_dir. bench.py's reference arm
    runs this in a child process, so the process that times the reference library never
    maps libnulpa.so."""
    import json
    import os
    dg, desc = build(name, scale, seed, device)
    g = dg.download()
    n, m2 = g.order(), g.directed_size()
    dg.free()
    os.makedirs(out_dir, exist_ok=True)
    g.offsets.tofile(os.path.join(out_dir, "offsets.u64"))
    g.targets.tofile(os.path.join(out_dir, "targets.u32"))
    meta = {**desc, "n": n, "m2": m2, "scale": scale, "seed": seed}
    with open(os.path.join(out_dir, "meta.json"), "w") as f:
        json.dump(meta, f)
    return meta


def _main(argv=None) -> int:
    import argparse
    ap = argparse.ArgumentParser(prog="python -m paper_2411_11468_b200.workloads")
    sub = ap.add_subparsers(dest="cmd", required=True)
    ex = sub.add_parser("export", help="write a workload's CSR as raw arrays")
    ex.add_argument("--workload", default="rmat", choices=["rmat", "grid", "web", "sbm"])
    ex.add_argument("--scale", type=int, default=27)
    ex.add_argument("--seed", type=int, default=1)
    ex.add_argument("--device", type=int, default=0)
    ex.add_argument("--out", required=True)
    a = ap.parse_args(argv)
    export_csr(a.workload, a.scale, a.seed, a.out, a.device)
    return 0


if __name__ == "__main__":
    raise SystemExit(_main())
