# r03u: closing check of the final tree: full GPU suite, smoke, config-2 bench (CPU leg included), config-5 bench
mkdir -p gpurun_out
python -c "from paper_2412_04980_b200 import _build; _build.build()" > gpurun_out/r03u_build.log 2>&1
timeout -s KILL 1800 python -m pytest tests -q -m gpu > gpurun_out/r03u_gpu_tests.log 2>&1; echo TESTS_EXIT $? >> gpurun_out/r03u_gpu_tests.log
timeout -s KILL 200 python __graft_entry__.py smoke > gpurun_out/r03u_smoke.log 2>&1; echo SMOKE_EXIT $? >> gpurun_out/r03u_smoke.log
timeout -s KILL 1500 python bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/r03u_bench_c2.json 2> gpurun_out/r03u_bench_c2.err
timeout -s KILL 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu > gpurun_out/r03u_bench_c5.json 2> gpurun_out/r03u_bench_c5.err
echo DONE
