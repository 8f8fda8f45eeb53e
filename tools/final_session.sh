#!/bin/bash
# Round-end measurement session: GPU tests, smoke, bench line + reference arm,
# every workload's line, ncu launch lists (time + DRAM bytes) of the default and
# the MFD workload, ncu --set full of k_tiles / k_recv / k_mfd_tiles, and the
# large-configuration parity tests with their printed drift / checks.  Usage: TAG
T=${1:-r02f}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi_$T.txt
timeout -s KILL 1800 python -m pytest tests -m gpu -q -rs -p no:cacheprovider > $O/gputest_$T.txt 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity_large.py -m gpu -q -s -p no:cacheprovider > $O/parity_large_$T.txt 2>&1
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$T.txt 2>&1
timeout -s KILL 400 python bench.py > $O/bench_$T.json 2> $O/bench_$T.err
timeout -s KILL 400 python bench.py --impl reference > $O/bench_ref_$T.json 2> $O/bench_ref_$T.err
for wl in dem1000 dem4000n2 ens64 dem1000fill dem4000fill dem1000mfd dem10000mfd; do
  timeout -s KILL 600 python bench.py --workload $wl > $O/bench_${T}_$wl.json 2> $O/bench_${T}_$wl.err
done
for wl in dem10000 dem10000mfd; do
  LEMGPU_EAGER=1 timeout -s KILL 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -c 400 --csv --log-file $O/launches_${T}_$wl.csv \
    python bench.py --workload $wl --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
done
LEMGPU_EAGER=1 timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:k_tiles -s 1 -c 1 \
  -o $O/ncu_full_${T}_k_tiles python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
LEMGPU_EAGER=1 timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:k_recv -s 1 -c 1 \
  -o $O/ncu_full_${T}_k_recv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
LEMGPU_EAGER=1 timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:k_mfd_tiles -s 4 -c 2 \
  -o $O/ncu_full_${T}_k_mfd_tiles python bench.py --workload dem10000mfd --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ls -la $O | tail -30
