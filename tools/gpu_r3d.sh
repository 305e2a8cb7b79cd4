# r03d: full GPU suite, smoke, config-2 bench (with the CPU leg), config-5 and config-4 benches
mkdir -p gpurun_out
timeout -s KILL 1800 python -m pytest tests -q -m gpu > gpurun_out/r03d_gpu_tests.log 2>&1; echo TESTS_EXIT $? >> gpurun_out/r03d_gpu_tests.log
timeout -s KILL 200 python __graft_entry__.py smoke > gpurun_out/r03d_smoke.log 2>&1; echo SMOKE_EXIT $? >> gpurun_out/r03d_smoke.log
timeout -s KILL 1500 python bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/r03d_bench_c2.json 2> gpurun_out/r03d_bench_c2.err
timeout -s KILL 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu > gpurun_out/r03d_bench_c5.json 2> gpurun_out/r03d_bench_c5.err
timeout -s KILL 900 python bench.py --config c4_40 --steps 2 --warmup 3 --no-cpu > gpurun_out/r03d_bench_c4_40.json 2> gpurun_out/r03d_bench_c4_40.err
timeout -s KILL 600 python bench.py --config c3_40 --steps 3 --warmup 3 --no-cpu > gpurun_out/r03d_bench_c3_40.json 2> gpurun_out/r03d_bench_c3_40.err
echo DONE
