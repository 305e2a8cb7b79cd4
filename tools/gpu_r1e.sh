# r01e validation: GPU tests, smoke, config-2 / config-5 bench, ncu capture of the strip kernels
set -x
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/r01e_gpu_tests.log 2>&1; echo TESTS_EXIT $? >> gpurun_out/r01e_gpu_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r01e_smoke.log 2>&1; echo SMOKE_EXIT $? >> gpurun_out/r01e_smoke.log
timeout 900 python bench.py > gpurun_out/r01e_bench_c2.json 2> gpurun_out/r01e_bench_c2.err
timeout 900 python bench.py --config c5 --steps 2 > gpurun_out/r01e_bench_c5.json 2> gpurun_out/r01e_bench_c5.err
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_r1w|k_resnorm|k_r1s' -f -o gpurun_out/r01e_targets python tools/ncu_targets.py c2 > gpurun_out/r01e_ncu.log 2>&1
echo done
