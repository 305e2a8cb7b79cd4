# r02u: resident GMRES neighbour flags + hierarchical last-arriver reductions (HDB_RES_FLAGS) A/B
mkdir -p gpurun_out
for fl in 0 1; do
  echo "== HDB_RES_FLAGS=$fl" >> gpurun_out/r02u_modes.log
  HDB_RES_FLAGS=$fl timeout -s KILL 300 python tools/gmres_modes.py c2 --levels 4,5,6,7 >> gpurun_out/r02u_modes.log 2>&1
done
for pts in 64 128 256; do
  echo "== HDB_RES_FLAGS=1 HDB_RES_GRID_PTS=$pts" >> gpurun_out/r02u_modes.log
  HDB_RES_GRID_PTS=$pts timeout -s KILL 300 python tools/gmres_modes.py c2 --levels 6,7 >> gpurun_out/r02u_modes.log 2>&1
done
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "device_resident or full_solve or config3 or presets or fgmres or vcycle or config1 or reproducible" > gpurun_out/r02u_focus.log 2>&1; echo FOCUS_EXIT $? >> gpurun_out/r02u_focus.log
timeout -s KILL 900 python bench.py --steps 3 --warmup 2 --no-cpu > gpurun_out/r02u_bench.json 2> gpurun_out/r02u_bench.err
echo DONE
