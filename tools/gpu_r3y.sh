# r03y: final tree: measured parity deltas of every configuration, ncu launch list of the config-5 solve
mkdir -p gpurun_out
timeout -s KILL 1800 python tools/parity_report.py --out gpurun_out/r03y_parity.json > gpurun_out/r03y_parity.log 2>&1
timeout -s KILL 400 python tools/profile_solve.py c5 --repeat 1 > gpurun_out/r03y_plain.log 2>&1 && \
timeout -s KILL 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r03y_launches_c5.csv python tools/profile_solve.py c5 --repeat 1 > gpurun_out/r03y_ncu.log 2>&1
echo DONE
