# r02y: fused residual+restriction (clamped window + per-lane closure overrides), per-size microbench, FRB sweep
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "fused_residual_restrict or folded_sum" > gpurun_out/r02y_focus.log 2>&1; echo FOCUS_EXIT $? >> gpurun_out/r02y_focus.log
for frb in 4 8; do
  echo "== HDB_RR_FRB=$frb" >> gpurun_out/r02y_fusion.log
  HDB_RR_FRB=$frb timeout -s KILL 300 python tools/fusion_bench.py >> gpurun_out/r02y_fusion.log 2>&1
done
timeout -s KILL 300 python tools/fusion_bench.py --sizes 2049 --reps 3 > gpurun_out/r02y_plain.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_resrestrict -c 2 -o gpurun_out/r02y_rr \
  python tools/fusion_bench.py --sizes 2049 --reps 3 > gpurun_out/r02y_ncu.log 2>&1
echo DONE
