# r03e: resident GMRES short-slice dots (all loads of a vector pair in flight) and 16-deep updates: cluster vs grid mode
mkdir -p gpurun_out
HDB_SMALL_N=150000 timeout -s KILL 300 python tools/gmres_modes.py c2 --levels 5,6,7 > gpurun_out/r03e_modes.log 2>&1
HDB_SMALL_N=150000 HDB_RES_SBASIS=0 timeout -s KILL 300 python tools/gmres_modes.py c2 --levels 6,7 > gpurun_out/r03e_modes_nosb.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "device_resident or full_solve or config3 or reproducible" > gpurun_out/r03e_focus.log 2>&1; echo FOCUS_EXIT $? >> gpurun_out/r03e_focus.log
echo DONE
