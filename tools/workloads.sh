#!/bin/bash
# Bench lines of every workload (device-resident value only) + a 2-rank run on one GPU (gloo).
for wl in dem1000 dem4000n2 ens64; do
  timeout -s KILL 300 python bench.py --workload $wl --no-cpu-baseline --e2e-steps 0 --steps 10 > gpurun_out/wl_$wl.json 2> gpurun_out/wl_$wl.err
  python -c "import json; d=json.load(open('gpurun_out/wl_$wl.json')); print('$wl', round(d['ms_per_step'],4), '%.3e' % d['value'], {k: round(v,4) for k,v in d['roofline']['kernel_ms'].items()})" || tail -3 gpurun_out/wl_$wl.err
done
LEMGPU_BENCH_BACKEND=gloo timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --workload ens64 --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/wl_ens64_2ranks.json 2> gpurun_out/wl_ens64_2ranks.err
python -c "import json; d=json.load(open('gpurun_out/wl_ens64_2ranks.json')); print('ens64 x2 ranks (gloo, 1 GPU)', d['n_gpus'], round(d['ms_per_step'],3), '%.3e' % d['value'])" || tail -5 gpurun_out/wl_ens64_2ranks.err
timeout -s KILL 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/ref_arm.json 2> gpurun_out/ref_arm.err; cat gpurun_out/ref_arm.json | head -c 600; echo
