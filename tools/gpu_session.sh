nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout -s KILL 1500 python -m pytest tests -m gpu -q -rs --durations=25 -p no:cacheprovider > gpurun_out/gputest_r02a.txt 2>&1
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02a.txt 2>&1
bash tools/profile_round.sh r02a
bash tools/workloads.sh r02a > gpurun_out/workloads_r02a.txt 2>&1
