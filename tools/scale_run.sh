#!/bin/bash
# Bench one config at several GPU counts (run on the GPU box).
# usage: tools/scale_run.sh CONFIG "1 2 4" [extra bench args]
cfg=$1; ns=$2; shift 2
mkdir -p gpurun_out
for n in $ns; do
  if [ "$n" = 1 ]; then
    timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu "$@" > gpurun_out/bench_${cfg}_n1.log 2>&1
  else
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + n)) bench.py --gpus $n --config $cfg --steps 10 --warmup 3 "$@" > gpurun_out/bench_${cfg}_n${n}.log 2>&1
  fi
  echo "$cfg n=$n rc=$?" >> gpurun_out/scale_status.txt
done
