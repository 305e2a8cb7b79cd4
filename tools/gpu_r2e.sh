# r02e: parity report (all configs with a reference record, both engine modes), full GPU suite, ncu of the TMA-ring MGS
mkdir -p gpurun_out
python -c "from paper_2412_04980_b200 import _build; _build.build()" > gpurun_out/r02e_build.log 2>&1
timeout -s KILL 1500 python tools/parity_report.py --out gpurun_out/r02e_parity.json > gpurun_out/r02e_parity.log 2>&1
timeout -s KILL 900 python -m pytest tests -q -m gpu > gpurun_out/r02e_gpu_tests.log 2>&1; echo TESTS_EXIT $? >> gpurun_out/r02e_gpu_tests.log
timeout -s KILL 300 python tools/mgs_target.py 12 > gpurun_out/r02e_mgs_plain.log 2>&1 && \
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_mgs -c 12 -o gpurun_out/r02e_mgs_ls python tools/mgs_target.py 12 > gpurun_out/r02e_ncu.log 2>&1
echo DONE
