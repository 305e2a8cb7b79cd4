# r03o: fault locator inside the sharded streaming low-sync step + sync floors
mkdir -p gpurun_out
for i in 1 2 3 4 5 6 7 8 9 10; do
  echo "== lsh-shard + HDB_DEBUG_SYNC run $i" >> gpurun_out/r03o.log
  HDB_LSH_SHARD_N=0 HDB_DEBUG_SYNC=1 timeout -s KILL 300 python tools/slab_sensitivity.py 2>&1 | grep -E "rel_delta|illegal|collectives|Error|after a|lsh fault" >> gpurun_out/r03o.log
done
bash tools/gpu_r3n.sh
echo DONE
