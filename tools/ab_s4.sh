# A/B of the S4 launch geometry (LMSCALE_S4_OCC CTAs/SM x LMSCALE_S4_GR rows per group)
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_step_parity.py -q -x > gpurun_out/t_step.log 2>&1; echo rc=$? >> gpurun_out/t_step.log
for c in ${CONFIGS:-1b tieba}; do
 for occ in ${OCCS:-2 3 4}; do for gr in ${GRS:-2 4 8}; do
  LMSCALE_NO_PDL=1 LMSCALE_S4_OCC=$occ LMSCALE_S4_GR=$gr timeout -s KILL 120 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e --no-dense > gpurun_out/ab/${c}_o${occ}_g${gr}.log 2>&1
 done; done
done
