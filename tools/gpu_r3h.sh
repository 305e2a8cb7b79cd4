# r03h: L2 eviction priorities in the hybrid MGS step (config 5 / config 4)
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "streaming_lowsync or lowsync" > gpurun_out/r03h_focus.log 2>&1; echo FOCUS_EXIT $? >> gpurun_out/r03h_focus.log
for h in 1 0; do
HDB_MGS2_HINT=$h timeout -s KILL 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu > gpurun_out/r03h_bench_c5_hint$h.json 2> gpurun_out/r03h_bench_c5_hint$h.err
done
timeout -s KILL 900 python bench.py --config c4_40 --steps 2 --warmup 3 --no-cpu > gpurun_out/r03h_bench_c4_40.json 2> gpurun_out/r03h_bench_c4_40.err
echo DONE
