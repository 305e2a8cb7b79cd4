# r02t: state check after the session restart: full GPU suite, smoke, bench, launch list
mkdir -p gpurun_out
python -c "from paper_2412_04980_b200 import _build; _build.build()" > gpurun_out/r02t_build.log 2>&1
timeout -s KILL 1200 python -m pytest tests -q -m gpu > gpurun_out/r02t_gpu_tests.log 2>&1; echo TESTS_EXIT $? >> gpurun_out/r02t_gpu_tests.log
timeout -s KILL 200 python __graft_entry__.py smoke > gpurun_out/r02t_smoke.log 2>&1; echo SMOKE_EXIT $? >> gpurun_out/r02t_smoke.log
timeout -s KILL 1200 python bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/r02t_bench.json 2> gpurun_out/r02t_bench.err
timeout -s KILL 300 python tools/profile_solve.py c2 --repeat 1 > gpurun_out/r02t_plain.log 2>&1 && \
timeout -s KILL 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02t_launches.csv python tools/profile_solve.py c2 --repeat 1 > gpurun_out/r02t_ncu.log 2>&1
echo DONE
