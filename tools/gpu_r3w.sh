# r03w: closing check of the final tree (Givens fused into k_mgs_ls): full GPU suite, smoke, config-2 bench with the CPU leg, launch list
mkdir -p gpurun_out
python -c "from paper_2412_04980_b200 import _build; _build.build()" > gpurun_out/r03w_build.log 2>&1
timeout -s KILL 1800 python -m pytest tests -q -m gpu > gpurun_out/r03w_gpu_tests.log 2>&1; echo TESTS_EXIT $? >> gpurun_out/r03w_gpu_tests.log
timeout -s KILL 200 python __graft_entry__.py smoke > gpurun_out/r03w_smoke.log 2>&1; echo SMOKE_EXIT $? >> gpurun_out/r03w_smoke.log
timeout -s KILL 1500 python bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/r03w_bench_c2.json 2> gpurun_out/r03w_bench_c2.err
timeout -s KILL 300 python tools/profile_solve.py c2 --repeat 1 > gpurun_out/r03w_plain.log 2>&1 && \
timeout -s KILL 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r03w_launches.csv python tools/profile_solve.py c2 --repeat 1 > gpurun_out/r03w_ncu.log 2>&1
timeout -s KILL 300 python tools/profile_solve.py c2 --repeat 1 > gpurun_out/r03w_plain2.log 2>&1 && \
timeout -s KILL 1500 ncu --set full --clock-control none --import-source on -k regex:k_mgs_ls -s 1200 -c 4 -o gpurun_out/r03w_mgs_ls python tools/profile_solve.py c2 --repeat 1 > gpurun_out/r03w_ncu2.log 2>&1
echo DONE
