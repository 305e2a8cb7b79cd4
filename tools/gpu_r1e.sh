# radius-3 Galerkin stencil: 2 vs 4 outputs per thread (HDB_RG_VO), config-2 level 3
timeout 600 python -m pytest tests -x -q -m gpu -k "operator" > gpurun_out/r1j_tests.log 2>&1; echo tests rc=$? >> gpurun_out/r1j_tests.log
for V in 2 4 2 4; do echo "vo=$V $(HDB_RG_VO=$V timeout 300 python tools/kernel_bench.py c2 --reps 30 2>/dev/null)" >> gpurun_out/r1j_kb_vo.txt; done
echo "c5 vo=4 $(HDB_RG_VO=4 timeout 300 python tools/kernel_bench.py c5 --reps 20 2>/dev/null)" >> gpurun_out/r1j_kb_vo.txt
