# r02h: batched T loads in the low-sync MGS; full GPU suite; microbench; bench with the CPU leg
mkdir -p gpurun_out
python -c "from paper_2412_04980_b200 import _build; _build.build()" > gpurun_out/r02h_build.log 2>&1
timeout -s KILL 300 python tools/galerkin_bench.py c2 > gpurun_out/r02h_galerkin.log 2>&1
timeout -s KILL 900 python -m pytest tests -q -m gpu > gpurun_out/r02h_gpu_tests.log 2>&1; echo TESTS_EXIT $? >> gpurun_out/r02h_gpu_tests.log
timeout -s KILL 200 python __graft_entry__.py smoke > gpurun_out/r02h_smoke.log 2>&1; echo SMOKE_EXIT $? >> gpurun_out/r02h_smoke.log
timeout -s KILL 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/r02h_bench.json 2> gpurun_out/r02h_bench.err
echo DONE
