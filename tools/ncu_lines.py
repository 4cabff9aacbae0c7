"""Warp-stall samples aggregated per CUDA source line (file:line) for one
kernel of an ncu report (needs -lineinfo and --import-source on)."""
import collections
import csv
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{pat}"], capture_output=True, text=True).stdout
agg = collections.Counter()
text = {}
fname = "?"
hdr = None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        hdr = None
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("Function Name",):
        continue
    try:
        s = float(r[4] or 0)
    except (ValueError, IndexError):
        continue
    key = f"{fname}:{r[0]}"
    agg[key] += s
    text.setdefault(key, r[1].strip())
tot = sum(agg.values()) or 1
for k, v in agg.most_common(n):
    print(f"{v / tot * 100:5.1f}%  {k:18s} {text[k][:100]}")
