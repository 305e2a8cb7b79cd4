#!/bin/bash
# GMRES engine mode sweep with both orthogonalisations (GPU box)
for o in cgs2 mgs; do
  HDB_ORTHO=$o python tools/gmres_modes.py c2 > gpurun_out/modes_c2_$o.txt 2>&1
  HDB_ORTHO=$o python tools/gmres_modes.py c3_40 > gpurun_out/modes_c3_$o.txt 2>&1
done
