# r02g: resident grid size sweep; focused tests after removing the slower forms; bench
mkdir -p gpurun_out
python -c "from paper_2412_04980_b200 import _build; _build.build()" > gpurun_out/r02g_build.log 2>&1
for p in 0 4096 2048 1024 512 256; do
  echo "== HDB_RES_GRID_PTS=$p" >> gpurun_out/r02g_modes.log
  HDB_RES_GRID_PTS=$p timeout -s KILL 300 python tools/gmres_modes.py c2 --levels 4,5,6,7 >> gpurun_out/r02g_modes.log 2>&1
done
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "separable or lowsync or exact or bitexact or config2_analogue or full_solve or device_resident or config3 or config1" > gpurun_out/r02g_focus.log 2>&1; echo FOCUS_EXIT $? >> gpurun_out/r02g_focus.log
timeout -s KILL 900 python bench.py --steps 3 --warmup 2 --no-cpu > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err
echo DONE
