# r03x: one-iteration FGMRES: scalar update and finiteness guard folded into the reduction launches, cached pointer table;
# A/B, then the closing check of the final tree (full GPU suite, smoke, config-2 bench with the CPU leg, config 5)
mkdir -p gpurun_out
HDB_STEP1_FUSE=0 timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r03x_bench_off.json 2> gpurun_out/r03x_bench_off.err
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r03x_bench_on.json 2> gpurun_out/r03x_bench_on.err
timeout -s KILL 1800 python -m pytest tests -q -m gpu > gpurun_out/r03x_gpu_tests.log 2>&1; echo TESTS_EXIT $? >> gpurun_out/r03x_gpu_tests.log
timeout -s KILL 200 python __graft_entry__.py smoke > gpurun_out/r03x_smoke.log 2>&1; echo SMOKE_EXIT $? >> gpurun_out/r03x_smoke.log
timeout -s KILL 1500 python bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/r03x_bench_c2.json 2> gpurun_out/r03x_bench_c2.err
timeout -s KILL 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu > gpurun_out/r03x_bench_c5.json 2> gpurun_out/r03x_bench_c5.err
echo DONE
