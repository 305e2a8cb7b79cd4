# r02f: producer fixes in the low-sync MGS ring, column-marching K2, resident separable stencil
mkdir -p gpurun_out
python -c "from paper_2412_04980_b200 import _build; _build.build()" > gpurun_out/r02f_build.log 2>&1
timeout -s KILL 300 python tools/galerkin_bench.py c2 > gpurun_out/r02f_galerkin.log 2>&1
timeout -s KILL 600 python tools/gmres_modes.py c2 --levels 4,5,6,7 > gpurun_out/r02f_modes.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "separable or lowsync or exact or bitexact or config2_analogue or full_solve or device_resident or config3 or config1" > gpurun_out/r02f_focus.log 2>&1; echo FOCUS_EXIT $? >> gpurun_out/r02f_focus.log
timeout -s KILL 900 python bench.py --steps 3 --warmup 2 --no-cpu > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err
echo DONE
