# Jacobi strip kernel at 6 vs 5 CTAs/SM (HDB_R1_J6), config-2 and config-5 fine grids; c5 bench of the final tree
timeout -s KILL 600 python -m pytest tests -x -q -m gpu -k "strip or jacobi" > gpurun_out/r1m_tests.log 2>&1; echo rc=$? >> gpurun_out/r1m_tests.log
HDB_R1_J6=1 timeout -s KILL 600 python -m pytest tests -x -q -m gpu -k "strip or jacobi" >> gpurun_out/r1m_tests.log 2>&1; echo rc6=$? >> gpurun_out/r1m_tests.log
for J in 0 1 0 1; do echo "j6=$J $(HDB_R1_J6=$J timeout -s KILL 300 python tools/kernel_bench.py c2 --reps 30 2>/dev/null)" >> gpurun_out/r1m_kb.txt; done
timeout -s KILL 900 python bench.py --config c5 --steps 2 > gpurun_out/r01e2_bench_c5.json 2> gpurun_out/r01e2_bench_c5.err
echo "c5 j6=1 $(HDB_R1_J6=1 timeout -s KILL 300 python tools/kernel_bench.py c5 --reps 20 2>/dev/null)" >> gpurun_out/r1m_kb.txt
