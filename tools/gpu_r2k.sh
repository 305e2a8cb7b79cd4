# r02k: HBM-streaming low-sync MGS on the fine level
mkdir -p gpurun_out
python -c "from paper_2412_04980_b200 import _build; _build.build()" > gpurun_out/r02k_build.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "lowsync or full_solve or config2 or fgmres or config1" > gpurun_out/r02k_focus.log 2>&1; echo FOCUS_EXIT $? >> gpurun_out/r02k_focus.log
timeout -s KILL 900 python bench.py --steps 3 --warmup 2 --no-cpu > gpurun_out/r02k_bench.json 2> gpurun_out/r02k_bench.err
timeout -s KILL 1500 python tools/parity_report.py --cases c2,c2a,c4_h12_f40 --out gpurun_out/r02k_parity.json > gpurun_out/r02k_parity.log 2>&1
echo DONE
