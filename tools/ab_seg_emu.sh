#!/bin/bash
# A/B of the S4 launch geometry in the local-slot layout (G > 1, no S6 fold),
# timed by ncu per k_seg launch inside the one-GPU emulated step.
mkdir -p gpurun_out/abseg
for c in $CONFIGS; do
  for og in $GEOMS; do
    o=${og%x*}; g=${og#*x}
    if [ "$o" = 0 ]; then unset LMSCALE_S4_OCC LMSCALE_S4_GR; else export LMSCALE_S4_OCC=$o LMSCALE_S4_GR=$g; fi
    timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_seg \
      python tools/emu_profile.py $c 2 4 > gpurun_out/abseg/${c}_$og.csv 2>/dev/null
    python - "$c" "$og" gpurun_out/abseg/${c}_$og.csv <<'PY'
import csv, sys, statistics
rows = [r for r in csv.reader(open(sys.argv[3])) if len(r) > 10 and r[0].isdigit()]
v = [float(r[-1]) for r in rows][2:]   # skip the first step's two launches
print(sys.argv[1], sys.argv[2], "k_seg median us", round(statistics.median(v) / 1e3, 1), "n", len(v))
PY
  done
done
