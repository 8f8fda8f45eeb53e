LEMGPU_BENCH_BACKEND=gloo timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 5 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/b2.json 2> gpurun_out/b2.err
python -c "import json; d=json.load(open('gpurun_out/b2.json')); print(d['n_gpus'], d['ms_per_step'], '%.3e'%d['value'], d['config'], d['details'].get('parallelism'), d['details'].get('collective'), d['e2e']['value'])" || tail -20 gpurun_out/b2.err
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/b2ref.json 2> gpurun_out/b2ref.err
cat gpurun_out/b2ref.json | head -c 600; echo
