#!/bin/bash
# Round-end single-GPU evidence, run on the GPU box from the repo root:
# bench lines (headline + supporting + reference arm), ncu launch lists and
# full captures of the world-1 kernels, the GPU test suite and smoke().
set -u
O=gpurun_out/final
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > $O/g1_bench_tieba_1b.json 2> $O/g1_bench.err
timeout 900 python bench.py --steps 20 --warmup 5 --supporting amazon,char --no-cpu \
  > $O/g1_bench_tieba_supporting.json 2> $O/g1_bench_sup.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/g1_bench_reference.json 2> $O/g1_ref.err
for c in 1b tieba; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python tools/prof_step.py --config $c --steps 2 --warmup 2 --no-graph > $O/ncu_launches_$c.csv 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_seg|k_group' -s 2 -c 2 \
    -o $O/full_$c python tools/prof_step.py --config $c --steps 1 --warmup 1 --no-graph > $O/ncu_full_$c.log 2>&1
  python tools/ncu_raw.py $O/full_$c.ncu-rep --csv > $O/ncu_full_$c.csv
  python tools/ncu_lines.py $O/full_$c.ncu-rep k_group 25 > $O/ncu_lines_k_group_$c.txt
  python tools/ncu_lines.py $O/full_$c.ncu-rep k_seg 25 > $O/ncu_lines_k_seg_$c.txt
done
timeout 1500 python -m pytest tests -m gpu -q > $O/g1_pytest_gpu.log 2>&1
echo done > $O/status
