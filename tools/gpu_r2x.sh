# r02x: fused MG residual+restriction, r + t folded into the last post-smooth, R factor in shared memory
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "fused_residual_restrict or folded_sum or strip_kernels or vcycle or device_resident or fgmres_vs or full_solve" > gpurun_out/r02x_focus.log 2>&1; echo FOCUS_EXIT $? >> gpurun_out/r02x_focus.log
for rs in 0 1; do
  echo "== HDB_RES_RSM=$rs" >> gpurun_out/r02x_modes.log
  HDB_RES_RSM=$rs timeout -s KILL 300 python tools/gmres_modes.py c2 --levels 4,5,6,7 >> gpurun_out/r02x_modes.log 2>&1
done
HDB_FUSE_RR=0 HDB_FUSE_RT=0 HDB_RES_RSM=0 timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r02x_bench_off.json 2> gpurun_out/r02x_bench_off.err
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r02x_bench_on.json 2> gpurun_out/r02x_bench_on.err
echo DONE
