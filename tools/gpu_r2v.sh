# r02v: resident reductions A/B (0: one-phase, 1: padded flags + last-arriver, 2: two-phase), k_mgs_ls L2 hint sweep
mkdir -p gpurun_out
for fl in 0 1 2 3; do
  echo "== HDB_RES_FLAGS=$fl" >> gpurun_out/r02v_modes.log
  HDB_RES_FLAGS=$fl timeout -s KILL 300 python tools/gmres_modes.py c2 --levels 5,6,7 >> gpurun_out/r02v_modes.log 2>&1
done
for k in 5 -1 0 3 8 20; do
  HDB_LS_KEEP=$k timeout -s KILL 300 python tools/mgs_ls_sweep.py >> gpurun_out/r02v_ls.log 2>&1
done
echo DONE
