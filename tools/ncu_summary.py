"""Summaries for profiles/: a launch list (ncu --metrics gpu__time_duration.sum CSV) and a
--set full report (.ncu-rep), as plain text.
usage: python tools/ncu_summary.py launches.csv full.ncu-rep > profiles/<round>_ncu_summary.txt"""
import collections
import csv
import subprocess
import sys


def clean(name):
    """Kernel names as 'k_team<0, float, 0, 256, ...>' whatever ncu's name base."""
    return name.replace("(int)", "").replace("(bool)", "").replace("nulpa::dev::", "").replace(
        "nulpa::<unnamed>::", "")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h, rows = rows[0], rows[1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows:
        k = clean(r[ki]).split("(")[0]
        v = float(r[vi].replace(",", ""))
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(t for _, t in agg.values())
    print(f"== launch list ({path.split('/')[-1]}): {sum(c for c, _ in agg.values())} launches, "
          f"{tot / 1e6:.1f} ms total (cold-cache, serialised under ncu)")
    print(f"{'ms':>10} {'share':>6} {'count':>6}  kernel")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:30]:
        print(f"{t / 1e6:10.2f} {t / tot * 100:5.1f}% {c:6d}  {k[:90]}")


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
           "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
STALLS = ["long_scoreboard", "short_scoreboard", "wait", "branch_resolving", "barrier",
          "mio_throttle", "lg_throttle", "membar", "no_instruction", "math_pipe_throttle"]


def num(d, k):
    try:
        return float(d[k].replace(",", ""))
    except (KeyError, ValueError):
        return float("nan")


def ratio(d, a, b):
    den = num(d, b)
    return num(d, a) / den if den else float("nan")


def full(path):
    ms = METRICS + [f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio" for s in STALLS]
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", ",".join(ms)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units, data = rows[0], rows[1], rows[2:]
    print(f"\n== ncu --set full ({path.split('/')[-1]})")
    print("kernel | ms | DRAM rd GB | DRAM wr GB | DRAM %peak | L2 hit % | warps active % | "
          "issue active % | warp-inst (G) | ld sectors/req | smem bank conflicts (G) | "
          "top stalls (cycles per issue)")
    for r in data:
        d = dict(zip(h, r))
        u = dict(zip(h, units))

        def gb(k):
            v = float(d[k])
            return v / 1e3 if u[k] == "Mbyte" else v if u[k] == "Gbyte" else v / 1e9
        st = sorted(((float(d[f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"]), s)
                     for s in STALLS), reverse=True)[:4]
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
                 "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}.get(
            u.get("gpu__time_duration.sum", "msecond"), 1.0)  # -> ms
        print(f"{clean(d['Kernel Name']).split('(')[0][:58]} | {float(d['gpu__time_duration.sum']) * scale:.2f} | "
              f"{gb('dram__bytes_read.sum'):.2f} | {gb('dram__bytes_write.sum'):.2f} | "
              f"{float(d.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "nan") or "nan"):.1f} | "
              f"{float(d['lts__t_sector_hit_rate.pct']):.1f} | "
              f"{float(d['sm__warps_active.avg.pct_of_peak_sustained_active']):.1f} | "
              f"{float(d['smsp__issue_active.avg.pct_of_peak_sustained_active']):.1f} | "
              f"{float(d['smsp__inst_executed.sum']) / 1e9:.2f} | "
              f"{ratio(d, 'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum', 'l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum'):.2f} | "
              f"{num(d, 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum') / 1e9:.2f} | "
              + " ".join(f"{s}={v:.1f}" for v, s in st))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        if p.endswith(".csv"):
            launches(p)
        else:
            full(p)
