# r01 closing check: the tree as rebuilt in a fresh container — GPU tests, smoke, config-2 bench
timeout -s KILL 600 python -m pytest tests -q -m gpu > gpurun_out/r01g_gpu_tests.log 2>&1; echo TESTS_EXIT $? >> gpurun_out/r01g_gpu_tests.log
timeout -s KILL 200 python __graft_entry__.py smoke > gpurun_out/r01g_smoke.log 2>&1; echo SMOKE_EXIT $? >> gpurun_out/r01g_smoke.log
timeout -s KILL 400 python bench.py > gpurun_out/r01g_bench_c2.json 2> gpurun_out/r01g_bench_c2.err
