# r03b: resident GMRES without the neighbour-flag experiment (reverted), R factor in shared memory; device setup tests
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "device_setup or device_built or device_resident or full_solve or config3" > gpurun_out/r03b_focus.log 2>&1; echo FOCUS_EXIT $? >> gpurun_out/r03b_focus.log
timeout -s KILL 300 python tools/gmres_modes.py c2 --levels 4,5,6,7 > gpurun_out/r03b_modes.log 2>&1
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r03b_bench.json 2> gpurun_out/r03b_bench.err
echo DONE
