#!/bin/bash
# One GPU session of measurements for profiles/: the bench line, the ncu
# launch list of the same command (cold, serialised: shares only), and one
# `ncu --set full` capture of the dominant kernel.  Usage: tools/profile_round.sh TAG
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
timeout -s KILL 400 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
LEMGPU_EAGER=1 timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -c 400 --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $OUT/launches_$TAG.log 2>&1
LEMGPU_EAGER=1 timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:k_tiles -s 1 -c 1 \
  -o $OUT/ncu_full_$TAG python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $OUT/ncu_full_$TAG.log 2>&1
LEMGPU_EAGER=1 timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:k_recv -s 1 -c 1 \
  -o $OUT/ncu_recv_$TAG python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $OUT/ncu_recv_$TAG.log 2>&1
ls -la $OUT | tail -8
