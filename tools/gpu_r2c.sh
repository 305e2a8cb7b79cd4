# r02c: new kernels (low-sync MGS, separable K2): focused tests first, then the full GPU suite, bench, ncu of the MGS step
mkdir -p gpurun_out
python -c "from paper_2412_04980_b200 import _build; _build.build()" > gpurun_out/r02c_build.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "separable or lowsync or exact or bitexact" > gpurun_out/r02c_focus.log 2>&1; echo FOCUS_EXIT $? >> gpurun_out/r02c_focus.log
timeout -s KILL 900 python -m pytest tests -q -m gpu > gpurun_out/r02c_gpu_tests.log 2>&1; echo TESTS_EXIT $? >> gpurun_out/r02c_gpu_tests.log
timeout -s KILL 900 python bench.py --steps 3 --warmup 2 --no-model-check > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err
timeout -s KILL 300 python tools/mgs_target.py 12 > gpurun_out/r02c_mgs_plain.log 2>&1 && \
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_mgs -c 12 -o gpurun_out/r02c_mgs_ls python tools/mgs_target.py 12 > gpurun_out/r02c_ncu.log 2>&1
echo DONE
