# launch list (per-kernel durations, DRAM bytes) of one eager step of a workload: tools/ncu_launches.sh WORKLOAD TAG
wl=$1; tag=$2
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${tag}_$wl.csv python bench.py --workload $wl --steps 1 --warmup 3 --e2e-steps 0 \
  --no-cpu-baseline --options '{"eager": 1}' > gpurun_out/launches_${tag}_$wl.log 2>&1
python tools/launch_summary.py gpurun_out/launches_${tag}_$wl.csv 1 > gpurun_out/launches_${tag}_$wl.txt 2>&1
