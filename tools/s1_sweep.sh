#!/bin/bash
# S1 grid-size sweep at world 1: tools/s1_sweep.sh "CFG..." "CTAS..."
# per (config, grid): the in-kernel phase trace of a few eager steps and a
# short bench line (graph replay, L2 flushed) -> gpurun_out/s1/
cfgs=${1:-"1b tieba"}; ctas=${2:-"148 96 74 48 32"}
mkdir -p gpurun_out/s1
for c in $cfgs; do
  for n in $ctas; do
    LMSCALE_S1_CTAS=$n LMSCALE_PHASE_TRACE=1 TRACE_NO_EVENTS=1 timeout 300 \
      python tools/trace_step.py $c 6 > gpurun_out/s1/trace_${c}_${n}.log 2>&1
    LMSCALE_S1_CTAS=$n timeout 300 python bench.py --config $c --supporting none --no-e2e \
      --no-cpu --steps 20 --warmup 5 > gpurun_out/s1/bench_${c}_${n}.json 2> gpurun_out/s1/bench_${c}_${n}.err
    echo "$c $n rc=$?" >> gpurun_out/s1/status
  done
done
