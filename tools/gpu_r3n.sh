# r03n: synchronisation floors (grid barrier / reductions over all SMs, cluster all-gathers) beside the resident per-iteration times
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/grid_sync tools/ubench/grid_sync.cu > gpurun_out/r03n_build.log 2>&1 && /tmp/grid_sync > gpurun_out/r03n_sync_floors.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/reduce_step tools/ubench/reduce_step.cu >> gpurun_out/r03n_build.log 2>&1 && /tmp/reduce_step >> gpurun_out/r03n_sync_floors.log 2>&1
timeout -s KILL 300 python tools/gmres_modes.py c2 --levels 4,5,6,7 > gpurun_out/r03n_modes.log 2>&1
echo DONE
