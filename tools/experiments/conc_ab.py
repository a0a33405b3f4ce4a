"""A/B of NULPA_CONCURRENT (side-by-side tier groups) on one workload, unprofiled runs.

usage: python tools/experiments/conc_ab.py WORKLOAD [SCALE] [RUNS]
Runs itself once per mode in a child process (the switch is read once per process) and
prints loop ms per run (median), iterations and modularity of the last run.
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def child(name: str, scale: int, runs: int) -> None:
    import numpy as np
    import torch

    from paper_2411_11468_b200 import labelprop as lp, workloads

    dg, _ = workloads.build(name, scale=scale, seed=1)
    cfg = lp.LpaConfig()
    out = torch.empty(dg.n, dtype=torch.int32, device="cuda:0")
    ms, qs, its = [], [], []
    for r in range(runs + 3):
        res = dg.lpa(cfg, labels_device_ptr=out.data_ptr(), want_host=False)
        if r >= 3:
            ms.append(res.stats.elapsed_seconds * 1e3)
            its.append(res.stats.iterations)
            qs.append(dg.modularity_device(out.data_ptr()))
    print(f"{name}{scale if name == 'rmat' else ''} {os.environ.get('CONC_TAG')}: "
          f"loop median {np.median(ms):.3f} ms (min {min(ms):.3f}) iters {sorted(set(its))} "
          f"Q mean {np.mean(qs):.4f} min {min(qs):.4f}", flush=True)


if __name__ == "__main__":
    name = sys.argv[1]
    scale = int(sys.argv[2]) if len(sys.argv) > 2 else 27
    runs = int(sys.argv[3]) if len(sys.argv) > 3 else 10
    if os.environ.get("CONC_CHILD"):
        child(name, scale, runs)
    else:
        # each token: MODE[,VAR=VALUE...] (extra switches for that child)
        for tok in os.environ.get("CONC_MODES", "0 1").split():
            mode, *extra = tok.split(",")
            env = dict(os.environ, NULPA_CONCURRENT=mode, CONC_CHILD="1")
            env.update(x.split("=", 1) for x in extra)
            env["CONC_TAG"] = tok
            subprocess.run([sys.executable, __file__, name, str(scale), str(runs)], env=env,
                           timeout=900)
