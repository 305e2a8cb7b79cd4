# r02l: persistent K2 tiles; low-sync HBM step with one all-reduce per reduction on sharded levels
mkdir -p gpurun_out
python -c "from paper_2412_04980_b200 import _build; _build.build()" > gpurun_out/r02l_build.log 2>&1
timeout -s KILL 300 python tools/galerkin_bench.py c2 > gpurun_out/r02l_galerkin.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_distributed.py tests/test_gpu_parity.py -q -m gpu -x -k "slab or separable or lowsync or full_solve or config2_analogue or bitexact" > gpurun_out/r02l_focus.log 2>&1; echo FOCUS_EXIT $? >> gpurun_out/r02l_focus.log
timeout -s KILL 900 python bench.py --steps 3 --warmup 2 --no-cpu > gpurun_out/r02l_bench.json 2> gpurun_out/r02l_bench.err
echo DONE
