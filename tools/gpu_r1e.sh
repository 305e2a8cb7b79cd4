# r01e final validation of the committed tree: GPU tests, smoke, config-2 bench (with cpu_baseline)
timeout -s KILL 900 python -m pytest tests -q -m gpu > gpurun_out/r01e3_gpu_tests.log 2>&1; echo TESTS_EXIT $? >> gpurun_out/r01e3_gpu_tests.log
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/r01e3_smoke.log 2>&1; echo SMOKE_EXIT $? >> gpurun_out/r01e3_smoke.log
timeout -s KILL 900 python bench.py > gpurun_out/r01e3_bench_c2.json 2> gpurun_out/r01e3_bench_c2.err
