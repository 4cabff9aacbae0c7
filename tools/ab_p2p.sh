# A/B of the fused S5+S6 P2P kernel at G = $N: CTAs per SM, and the warp-load kernel
mkdir -p gpurun_out/abp
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/abp/build.log 2>&1
for cps in 1 2 3 4; do
  LMSCALE_P2P_CTAS_PER_SM=$cps timeout -s KILL 600 python bench.py --gpus $N --no-e2e --no-cpu --no-dense --steps 10 > gpurun_out/abp/g${N}_cps$cps.log 2>&1
done
LMSCALE_NO_P2P_BULK=1 timeout -s KILL 600 python bench.py --gpus $N --no-e2e --no-cpu --no-dense --steps 10 > gpurun_out/abp/g${N}_old.log 2>&1
