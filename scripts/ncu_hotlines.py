"""Warp-stall samples per CUDA source line for one kernel launch of an ncu report
(needs -lineinfo and --import-source).  Used to pick what to optimise.
usage: python scripts/ncu_hotlines.py REPORT KERNEL_REGEX [TOP] [LAUNCH_SKIP]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre, "--launch-skip", skip,
                      "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows, fname, hdr = [], "", None
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = r
    elif r[0].isdigit() and hdr:
        try:
            s, ns, ins = int(r[4] or 0), int(r[5] or 0), int(r[7] or 0)
        except ValueError:
            continue
        rows.append((s, ns, ins, f"{fname}:{r[0]}", r[1].strip()[:110]))
tot = sum(x[0] for x in rows) or 1
print(f"total stall samples {tot}")
for s, ns, ins, loc, src in sorted(rows, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}% (not-issued {100 * ns / tot:5.1f}%) inst={ins:>10d} {loc:18s} {src}")
