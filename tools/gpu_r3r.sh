# r03r: after the tile-sampling fix: sharded streaming low-sync step stress (was ~40 % faults), distributed + Galerkin tests
mkdir -p gpurun_out
for i in 1 2 3 4 5 6 7 8 9 10; do
  echo "== lsh-shard run $i" >> gpurun_out/r03r.log
  HDB_LSH_SHARD_N=0 timeout -s KILL 300 python tools/slab_sensitivity.py 2>&1 | grep -E "rel_delta|illegal|collectives|Error|after a|lsh fault" >> gpurun_out/r03r.log
done
for i in 1 2 3 4; do
  echo "== lsh-shard + HDB_DEBUG_SYNC run $i" >> gpurun_out/r03r.log
  HDB_LSH_SHARD_N=0 HDB_DEBUG_SYNC=1 timeout -s KILL 300 python tools/slab_sensitivity.py 2>&1 | grep -E "rel_delta|illegal|collectives|Error|after a|lsh fault" >> gpurun_out/r03r.log
done
HDB_LSH_SHARD_N=0 timeout -s KILL 1200 python -m pytest tests/test_gpu_distributed.py -q -m gpu -x > gpurun_out/r03r_dist_lsh.log 2>&1; echo DIST_EXIT $? >> gpurun_out/r03r_dist_lsh.log
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "operator or galerkin or separable or transfers" > gpurun_out/r03r_ops.log 2>&1; echo OPS_EXIT $? >> gpurun_out/r03r_ops.log
echo DONE
