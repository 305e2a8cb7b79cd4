# r03l: measured parity deltas (all configurations incl. the reduced config 5), full GPU suite, smoke, config-2 bench with the CPU leg, launch list
mkdir -p gpurun_out
timeout -s KILL 1800 python tools/parity_report.py --out gpurun_out/r03l_parity.json > gpurun_out/r03l_parity.log 2>&1
timeout -s KILL 1800 python -m pytest tests -q -m gpu > gpurun_out/r03l_gpu_tests.log 2>&1; echo TESTS_EXIT $? >> gpurun_out/r03l_gpu_tests.log
timeout -s KILL 200 python __graft_entry__.py smoke > gpurun_out/r03l_smoke.log 2>&1; echo SMOKE_EXIT $? >> gpurun_out/r03l_smoke.log
timeout -s KILL 1500 python bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/r03l_bench_c2.json 2> gpurun_out/r03l_bench_c2.err
timeout -s KILL 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu > gpurun_out/r03l_bench_c5.json 2> gpurun_out/r03l_bench_c5.err
timeout -s KILL 300 python tools/profile_solve.py c2 --repeat 1 > gpurun_out/r03l_plain.log 2>&1 && \
timeout -s KILL 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r03l_launches.csv python tools/profile_solve.py c2 --repeat 1 > gpurun_out/r03l_ncu.log 2>&1
echo DONE
