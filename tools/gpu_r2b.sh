# r02b: GPU tests after the launch-accounting change, the new bench, one ncu capture of the MGS step
mkdir -p gpurun_out
python -c "from paper_2412_04980_b200 import _build; _build.build()" > gpurun_out/r02b_build.log 2>&1
timeout -s KILL 900 python -m pytest tests -q -m gpu -x > gpurun_out/r02b_gpu_tests.log 2>&1; echo TESTS_EXIT $? >> gpurun_out/r02b_gpu_tests.log
timeout -s KILL 900 python bench.py --steps 3 --warmup 2 > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err
timeout -s KILL 300 python tools/profile_solve.py c2 --repeat 1 > gpurun_out/r02b_plain.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_mgs_grid -s 300 -c 3 -o gpurun_out/r02b_mgs python tools/profile_solve.py c2 --repeat 1 > gpurun_out/r02b_ncu.log 2>&1
echo DONE
