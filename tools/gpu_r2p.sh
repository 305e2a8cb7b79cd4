mkdir -p gpurun_out
python -c "from paper_2412_04980_b200 import _build; _build.build()" > gpurun_out/r02p_build.log 2>&1
timeout -s KILL 300 python tools/slab_sensitivity.py > gpurun_out/r02p_slab.log 2>&1
timeout -s KILL 300 python tools/slab_sensitivity.py > gpurun_out/r02p_slab2.log 2>&1
echo DONE
