#!/bin/bash
# ens64 at N=1 (the strong-scaling counterpart), dem10000, and the 2-rank path on one GPU (gloo rendezvous, no NCCL).
tag=${1:-ens}
timeout -s KILL 400 python bench.py --workload ens64 --no-cpu-baseline --e2e-steps 0 --steps 10 > gpurun_out/${tag}_ens64.json 2> gpurun_out/${tag}_ens64.err
python -c "import json; d=json.load(open('gpurun_out/${tag}_ens64.json')); print('ens64', round(d['ms_per_step'],4), '%.3e' % d['value'], d['roofline']['kernel_ms'], d['details']['member_stats'])" || tail -5 gpurun_out/${tag}_ens64.err
LEMGPU_BENCH_BACKEND=gloo timeout -s KILL 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${tag}_ens64_2ranks.json 2> gpurun_out/${tag}_ens64_2ranks.err
python -c "import json; d=json.load(open('gpurun_out/${tag}_ens64_2ranks.json')); print('default at 2 ranks (gloo, 1 GPU):', d['config']['workload'][:40], d['n_gpus'], round(d['ms_per_step'],3), '%.3e' % d['value'], d['scaling'])" || tail -5 gpurun_out/${tag}_ens64_2ranks.err
