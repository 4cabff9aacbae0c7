#!/bin/bash
# Round-end N-GPU evidence (N = 2 or 4), run on the GPU box from the repo root:
# bench lines (fp32 and compressed exchange) and the multi-GPU test suite.
set -u
N=$1
O=gpurun_out/final_g$N
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvidia-smi topo -m > $O/g${N}_topo.txt 2>&1
timeout 900 python bench.py --gpus $N --steps 20 --warmup 5 --supporting 1b,amazon \
  > $O/g${N}_bench_tieba_1b_amazon.json 2> $O/bench.err
timeout 900 python bench.py --gpus $N --steps 20 --warmup 5 --compress 1.0 --supporting 1b --no-e2e \
  > $O/g${N}_bench_tieba_compressed.json 2> $O/bench_c.err
timeout 1500 python -m pytest tests/test_multigpu.py -q -v > $O/g${N}_pytest_multigpu.log 2>&1
echo done > $O/status
