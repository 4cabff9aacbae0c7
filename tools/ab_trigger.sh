#!/bin/bash
# A/B of the early programmatic trigger of the world-1 S4 at small K:
# alternating bench lines (1b, 50 steps) with and without it, phase traces,
# and the world-1 step parity tests -> gpurun_out/trig/
# (historical: the LMSCALE_NO_EARLY_TRIGGER switch and the trigger itself were
# removed after this A/B showed no gain -- DESIGN.md, rejected table)
mkdir -p gpurun_out/trig
for rep in 1 2 3; do
  for tag in on off; do
    env=""; [ $tag = off ] && env="LMSCALE_NO_EARLY_TRIGGER=1"
    env $env timeout 300 python bench.py --config 1b --supporting none --no-e2e --no-cpu \
      --steps 50 --warmup 5 > gpurun_out/trig/bench_${tag}_${rep}.json 2>/dev/null
  done
done
for tag in on off; do
  env=""; [ $tag = off ] && env="LMSCALE_NO_EARLY_TRIGGER=1"
  env $env LMSCALE_PHASE_TRACE=1 TRACE_NO_EVENTS=1 timeout 300 python tools/trace_step.py 1b 6 \
    > gpurun_out/trig/trace_${tag}.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_step_parity.py tests/test_gpu_parity.py -q -x \
  > gpurun_out/trig/pytest.log 2>&1
echo done > gpurun_out/trig/status
