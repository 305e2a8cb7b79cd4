# r03s: final tree (slab tile-sampling fix, sharded low-sync step on by default): full GPU suite, smoke, config-2 bench, config 5
mkdir -p gpurun_out
timeout -s KILL 1800 python -m pytest tests -q -m gpu > gpurun_out/r03s_gpu_tests.log 2>&1; echo TESTS_EXIT $? >> gpurun_out/r03s_gpu_tests.log
timeout -s KILL 200 python __graft_entry__.py smoke > gpurun_out/r03s_smoke.log 2>&1; echo SMOKE_EXIT $? >> gpurun_out/r03s_smoke.log
timeout -s KILL 1500 python bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/r03s_bench_c2.json 2> gpurun_out/r03s_bench_c2.err
timeout -s KILL 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r03s_bench_reference_c2.json 2> gpurun_out/r03s_bench_reference_c2.err
for i in 1 2 3 4 5 6; do
  echo "== default run $i" >> gpurun_out/r03s_stress.log
  timeout -s KILL 300 python tools/slab_sensitivity.py 2>&1 | grep -E "rel_delta|illegal|collectives|Error|after a|lsh fault" >> gpurun_out/r03s_stress.log
done
echo DONE
