"""Print the hottest SASS lines (by warp stall samples) per kernel from an ncu report."""
import csv, subprocess, sys
rep, pat = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{pat}"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1], None, []]; blocks.append(cur); continue
    if cur is not None and cur[1] is None:
        cur[1] = r; continue
    if cur is not None and r:
        cur[2].append(r)
for name, hdr, body in blocks[:1]:
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_src = hdr.index("Source")
    tot = sum(float(r[i_s] or 0) for r in body)
    print(name[:80], "samples", tot)
    for r in sorted(body, key=lambda r: -float(r[i_s] or 0))[:n]:
        print(f"{float(r[i_s] or 0)/max(tot,1)*100:5.1f}%  {r[i_src][:110]}")
