# r03v: Givens / stopping update fused into the tail of k_mgs_ls (device-driven GMRES): parity focus + A/B
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "lowsync or config2_analogue or full_solve or reproducible or device_resident or config3 or presets or config5" > gpurun_out/r03v_focus.log 2>&1; echo FOCUS_EXIT $? >> gpurun_out/r03v_focus.log
HDB_LS_GIVENS=0 timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r03v_bench_off.json 2> gpurun_out/r03v_bench_off.err
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r03v_bench_on.json 2> gpurun_out/r03v_bench_on.err
echo DONE
