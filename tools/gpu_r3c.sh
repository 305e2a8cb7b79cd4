# r03c: rank-count-invariant reduction mode (row-ordered partials): P = 1, 2, 3, 4 thread-rank solves bit-identical
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_distributed.py -q -m gpu -x > gpurun_out/r03c_dist.log 2>&1; echo DIST_EXIT $? >> gpurun_out/r03c_dist.log
HDB_PINV=1 timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "full_solve or config3 or presets or bicgstab or vcycle or fgmres" > gpurun_out/r03c_pinv_parity.log 2>&1; echo PINV_EXIT $? >> gpurun_out/r03c_pinv_parity.log
echo DONE
