# ncu capture of k_esc_forest on the epsilon-filled 1000^2 DEM (eager launches)
N=${1:-1000}
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_esc_forest -s 1 -c 1 \
  -o gpurun_out/ncu_forest_$N python tools/forest_probe.py $N 2 eager=1 > gpurun_out/ncu_forest_$N.log 2>&1
ncu -i gpurun_out/ncu_forest_$N.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu_forest_src_$N.csv 2>/dev/null
python tools/ncu_srcprof.py gpurun_out/ncu_forest_src_$N.csv 40 > gpurun_out/ncu_forest_top_$N.txt
