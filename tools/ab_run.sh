#!/bin/bash
# A/B one multi-GPU config: tools/ab_run.sh CONFIG N TAG "ENV=VAL ..." [bench args]
cfg=$1; n=$2; tag=$3; envs=$4; shift 4
mkdir -p gpurun_out/ab
env $envs timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29700 + n)) bench.py --gpus $n --config $cfg --steps 10 --warmup 3 --no-e2e --no-dense "$@" > gpurun_out/ab/${cfg}_n${n}_${tag}.log 2>&1
echo "$cfg n=$n $tag rc=$?" >> gpurun_out/ab/status
