# r03f: streaming low-synchronisation MGS step on levels beyond the one-launch form (config 5 / config 4 level 3)
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "streaming_lowsync or lowsync or config2_analogue or full_solve" > gpurun_out/r03f_focus.log 2>&1; echo FOCUS_EXIT $? >> gpurun_out/r03f_focus.log
timeout -s KILL 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu > gpurun_out/r03f_bench_c5.json 2> gpurun_out/r03f_bench_c5.err
timeout -s KILL 900 python bench.py --config c4_40 --steps 2 --warmup 3 --no-cpu > gpurun_out/r03f_bench_c4_40.json 2> gpurun_out/r03f_bench_c4_40.err
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r03f_bench_c2.json 2> gpurun_out/r03f_bench_c2.err
echo DONE
