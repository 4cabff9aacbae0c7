"""Summarise key raw ncu metrics per kernel launch of a report.

    python tools/ncu_raw.py REPORT [--csv] [metric ...]
"""
import csv
import subprocess
import sys

args = [a for a in sys.argv[1:] if a != "--csv"]
as_csv = "--csv" in sys.argv
rep = args[0]
want = args[1:] or ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__registers_per_thread',
        'launch__grid_size', 'launch__block_size', 'launch__shared_mem_per_block_dynamic',
        'lts__t_bytes.sum',
        'smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_membar_per_issue_active.ratio']
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
cols = [w for w in want if w in hdr]
if as_csv:
    w = csv.writer(sys.stdout)
    w.writerow(["Kernel Name"] + cols)
    w.writerow(["(unit)"] + [rows[1][hdr.index(c)] for c in cols])
    for r in rows[2:]:
        w.writerow([r[hdr.index('Kernel Name')]] + [r[hdr.index(c)] for c in cols])
else:
    for r in rows[2:]:
        print(r[hdr.index('Kernel Name')][:60])
        for c in cols:
            print(f"   {c:75s} {r[hdr.index(c)]}")
