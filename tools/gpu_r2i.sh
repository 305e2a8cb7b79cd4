# r02i: batched resident reductions; modes; ncu of the roofline kernel inside the config-2 solve
mkdir -p gpurun_out
python -c "from paper_2412_04980_b200 import _build; _build.build()" > gpurun_out/r02i_build.log 2>&1
timeout -s KILL 300 python tools/gmres_modes.py c2 --levels 4,5,6,7 > gpurun_out/r02i_modes.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "device_resident or full_solve or config3 or presets or vcycle or fgmres" > gpurun_out/r02i_focus.log 2>&1; echo FOCUS_EXIT $? >> gpurun_out/r02i_focus.log
timeout -s KILL 900 python bench.py --steps 3 --warmup 2 --no-cpu > gpurun_out/r02i_bench.json 2> gpurun_out/r02i_bench.err
timeout -s KILL 300 python tools/profile_solve.py c2 --repeat 1 > gpurun_out/r02i_plain.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_mgs_ls -s 1200 -c 4 -o gpurun_out/r02i_mgs python tools/profile_solve.py c2 --repeat 1 > gpurun_out/r02i_ncu.log 2>&1
echo DONE
