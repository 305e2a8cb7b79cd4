# cooperative-MGS reductions: epoch flags (HDB_MGS_FLAGS=1) vs grid barrier (0); results must be bit-identical
timeout -s KILL 600 python -m pytest tests -x -q -m gpu -k "reproducible or analogue or resident or fgmres or preconditioner" > gpurun_out/r1l_tests.log 2>&1; echo tests rc=$? >> gpurun_out/r1l_tests.log
for F in 0 1 0 1; do HDB_MGS_FLAGS=$F timeout -s KILL 600 python bench.py --steps 3 --warmup 3 --no-cpu >> gpurun_out/r1l_bench_f$F.json 2>>gpurun_out/r1l_bench_f$F.err; done
