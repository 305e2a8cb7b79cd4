# r02s: resident basis slices in shared memory (HDB_RES_SBASIS) vs global
mkdir -p gpurun_out
python -c "from paper_2412_04980_b200 import _build; _build.build()" > gpurun_out/r02s_build.log 2>&1
for sb in 0 1; do
  echo "== HDB_RES_SBASIS=$sb" >> gpurun_out/r02s_modes.log
  HDB_RES_SBASIS=$sb timeout -s KILL 300 python tools/gmres_modes.py c2 --levels 4,5,6,7 >> gpurun_out/r02s_modes.log 2>&1
  HDB_RES_SBASIS=$sb timeout -s KILL 300 python tools/gmres_modes.py c3_40 --levels 5 >> gpurun_out/r02s_modes.log 2>&1
done
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "device_resident or full_solve or config3 or presets or fgmres or vcycle or config1" > gpurun_out/r02s_focus.log 2>&1; echo FOCUS_EXIT $? >> gpurun_out/r02s_focus.log
timeout -s KILL 900 python bench.py --steps 3 --warmup 2 --no-cpu > gpurun_out/r02s_bench.json 2> gpurun_out/r02s_bench.err
echo DONE
