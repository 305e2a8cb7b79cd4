# r02m: slab sensitivity (LS vs MGS order); resident LS-MGS (HDB_ORTHO=ls) vs DGKS
mkdir -p gpurun_out
python -c "from paper_2412_04980_b200 import _build; _build.build()" > gpurun_out/r02m_build.log 2>&1
timeout -s KILL 300 python tools/slab_sensitivity.py > gpurun_out/r02m_slab.log 2>&1
for o in dgks ls; do
  echo "== HDB_ORTHO=$o" >> gpurun_out/r02m_modes.log
  HDB_ORTHO=$o timeout -s KILL 300 python tools/gmres_modes.py c2 --levels 4,5,6,7 >> gpurun_out/r02m_modes.log 2>&1
done
HDB_ORTHO=ls timeout -s KILL 900 python tools/parity_report.py --cases c1s,wedge20,c2a,c3_40,c2 --out gpurun_out/r02m_parity_ls.json > gpurun_out/r02m_parity_ls.log 2>&1
HDB_ORTHO=ls timeout -s KILL 900 python bench.py --steps 3 --warmup 2 --no-cpu > gpurun_out/r02m_bench_ls.json 2> gpurun_out/r02m_bench_ls.err
echo DONE
