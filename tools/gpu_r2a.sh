# r02a: GPU tests of the round-1 tree, a short bench, then racecheck over the smem/TMA/cluster kernels
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -q -m gpu -x > gpurun_out/r02a_gpu_tests.log 2>&1; echo TESTS_EXIT $? >> gpurun_out/r02a_gpu_tests.log
timeout -s KILL 300 python tools/sanitize_targets.py > gpurun_out/r02a_sanitize_plain.log 2>&1; echo PLAIN_EXIT $? >> gpurun_out/r02a_sanitize_plain.log
timeout -s KILL 1500 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_targets.py > gpurun_out/r02a_racecheck.log 2>&1; echo RACECHECK_EXIT $? >> gpurun_out/r02a_racecheck.log
