# r03j: reduced config-5 parity (single GPU + two slabs), ncu capture of the hybrid MGS step inside the config-5 solve
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_distributed.py -q -m gpu -x -k "config5_reduced or nccl_binding" > gpurun_out/r03j_focus.log 2>&1; echo FOCUS_EXIT $? >> gpurun_out/r03j_focus.log
timeout -s KILL 300 python tools/profile_solve.py c5 --repeat 1 > gpurun_out/r03j_plain.log 2>&1 && \
timeout -s KILL 1500 ncu --set full --clock-control none --import-source on -k regex:k_mgs_grid2 -s 300 -c 3 -o gpurun_out/r03j_grid2 \
  python tools/profile_solve.py c5 --repeat 1 > gpurun_out/r03j_ncu.log 2>&1
echo DONE
