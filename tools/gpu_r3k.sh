# r03k: hybrid MGS step with 8 register slots and 16 basis loads per thread in flight
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "streaming_lowsync or lowsync" > gpurun_out/r03k_focus.log 2>&1; echo FOCUS_EXIT $? >> gpurun_out/r03k_focus.log
timeout -s KILL 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu > gpurun_out/r03k_bench_c5.json 2> gpurun_out/r03k_bench_c5.err
timeout -s KILL 900 python bench.py --config c4_40 --steps 2 --warmup 3 --no-cpu > gpurun_out/r03k_bench_c4_40.json 2> gpurun_out/r03k_bench_c4_40.err
echo DONE
