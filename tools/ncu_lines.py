"""Per-source-line hot spots of one kernel in an ncu report (--import-source on, -lineinfo):
    python tools/ncu_lines.py REPORT.ncu-rep [TOP]
Prints the source lines with the most warp-stall samples and executed warp instructions."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, path, hdr = [], None, None
for rec in csv.reader(io.StringIO(out)):
    if not rec:
        continue
    if rec[0] == "File Path":
        path = rec[1].split("/")[-1]
        continue
    if rec[0] == "Line No":
        hdr = rec
        continue
    if hdr is None or rec[0] in ("", "Function Name"):
        continue
    d = dict(zip(hdr[4:], rec[4:]))
    try:
        st, ins = int(d["Warp Stall Sampling (All Samples)"]), int(d["Instructions Executed"])
    except (KeyError, ValueError):
        continue
    rows.append((st, ins, f"{path}:{rec[0]}", rec[1][:110]))
tot_s = sum(r[0] for r in rows) or 1
tot_i = sum(r[1] for r in rows) or 1
print(f"total stall samples {tot_s}, warp instructions {tot_i}")
for st, ins, loc, src in sorted(rows, reverse=True)[:top]:
    print(f"{100 * st / tot_s:5.1f}% stall {100 * ins / tot_i:5.1f}% inst  {loc:24s} {src}")
