"""Per CUDA source line: warp-stall samples and instructions executed, from an
ncu --set full report (--import-source on), top N lines.

    python tools/ncu_lines.py <rep> <kernel-regex> [N]
"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern,
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows, fname = [], ""
hdr = None
for x in csv.reader(out.splitlines()):
    if x and x[0] == "File Path":
        fname = x[1].split("/")[-1]
        continue
    if x and x[0] == "Line No":
        hdr = x
        continue
    if hdr is None or len(x) != len(hdr) or not x[0]:
        continue
    try:
        rows.append((int(x[4] or 0), int(x[7] or 0), f"{fname}:{x[0]}", x[1].strip()[:80]))
    except ValueError:
        pass
tot = sum(r[0] for r in rows)
print(f"{kern}: {tot} stall samples, {sum(r[1] for r in rows)} instructions")
for s, n, loc, src in sorted(rows, key=lambda r: -r[0])[:top]:
    print(f"{s:6d} {100 * s / max(tot, 1):5.1f}% {n:10d}  {loc:16s} {src}")
