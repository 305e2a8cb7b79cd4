# r03t: device-driven GMRES on sharded levels (streaming low-sync step + in-stream all-reduces): distributed tests, stress
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests/test_gpu_distributed.py -q -m gpu -x > gpurun_out/r03t_dist.log 2>&1; echo DIST_EXIT $? >> gpurun_out/r03t_dist.log
HDB_GMRES_DEV_SHARD=0 timeout -s KILL 1500 python -m pytest tests/test_gpu_distributed.py -q -m gpu -x -k "heterogeneous or config5" > gpurun_out/r03t_dist_hostdriven.log 2>&1; echo DIST_EXIT $? >> gpurun_out/r03t_dist_hostdriven.log
for i in 1 2 3 4; do
  echo "== default run $i" >> gpurun_out/r03t_stress.log
  timeout -s KILL 300 python tools/slab_sensitivity.py 2>&1 | grep -E "rel_delta|single_its|slab_its|illegal|collectives|Error|after a|lsh fault" >> gpurun_out/r03t_stress.log
done
echo DONE
