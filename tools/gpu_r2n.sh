# r02n: pinned V-pointer mirror (illegal-access fix on sharded LS steps); auto resident ortho; full suite; bench
mkdir -p gpurun_out
python -c "from paper_2412_04980_b200 import _build; _build.build()" > gpurun_out/r02n_build.log 2>&1
timeout -s KILL 300 python tools/slab_sensitivity.py > gpurun_out/r02n_slab.log 2>&1
timeout -s KILL 900 python -m pytest tests -q -m gpu > gpurun_out/r02n_gpu_tests.log 2>&1; echo TESTS_EXIT $? >> gpurun_out/r02n_gpu_tests.log
timeout -s KILL 900 python bench.py --steps 3 --warmup 2 --no-cpu > gpurun_out/r02n_bench.json 2> gpurun_out/r02n_bench.err
echo DONE
