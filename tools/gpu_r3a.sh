# r03a: device-side setup tests, fused kernels, jacobi_add at 6 CTAs/SM, bench A/B of the fusions
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "device_setup or device_built or fused_residual_restrict or folded_sum or vcycle or full_solve" > gpurun_out/r03a_focus.log 2>&1; echo FOCUS_EXIT $? >> gpurun_out/r03a_focus.log
timeout -s KILL 300 python tools/fusion_bench.py > gpurun_out/r03a_fusion.log 2>&1
HDB_FUSE_RR=0 HDB_FUSE_RT=0 timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r03a_bench_off.json 2> gpurun_out/r03a_bench_off.err
HDB_FUSE_RT=0 timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r03a_bench_rr.json 2> gpurun_out/r03a_bench_rr.err
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r03a_bench_on.json 2> gpurun_out/r03a_bench_on.err
echo DONE
