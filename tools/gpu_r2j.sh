# r02j: L2 eviction hints in the low-sync MGS ring; grid-mode resident everywhere; tiny-launch costs
mkdir -p gpurun_out
python -c "from paper_2412_04980_b200 import _build; _build.build()" > gpurun_out/r02j_build.log 2>&1
timeout -s KILL 300 python tools/galerkin_bench.py c2 > gpurun_out/r02j_galerkin.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "device_resident or full_solve or config3 or presets or lowsync or config2_analogue" > gpurun_out/r02j_focus.log 2>&1; echo FOCUS_EXIT $? >> gpurun_out/r02j_focus.log
timeout -s KILL 900 python bench.py --steps 3 --warmup 2 --no-cpu > gpurun_out/r02j_bench.json 2> gpurun_out/r02j_bench.err
echo DONE
