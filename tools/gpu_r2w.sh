# r02w: ncu source-level capture of the resident GMRES on the 65^2 level (cluster and grid mode)
mkdir -p gpurun_out
HDB_SMALL_N=12000 timeout -s KILL 300 python tools/gmres_modes.py c2 --levels 7 --reps 1 > gpurun_out/r02w_plain.log 2>&1 && \
HDB_SMALL_N=12000 timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k regex:k_resident_gmres -c 6 \
  -o gpurun_out/r02w_res7 python tools/gmres_modes.py c2 --levels 7 --reps 1 > gpurun_out/r02w_ncu.log 2>&1
for sb in 0 1; do
  echo "== HDB_RES_SBASIS=$sb" >> gpurun_out/r02w_sbasis.log
  HDB_SMALL_N=12000 HDB_RES_SBASIS=$sb timeout -s KILL 300 python tools/gmres_modes.py c2 --levels 5,6,7 >> gpurun_out/r02w_sbasis.log 2>&1
done
echo DONE
