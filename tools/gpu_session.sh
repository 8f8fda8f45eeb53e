#!/bin/bash
# One GPU session: the GPU tests, smoke, the bench line + ncu launch list + ncu --set full
# of the dominant kernels, and every workload's bench line.  Usage: tools/gpu_session.sh TAG
T=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout -s KILL 1800 python -m pytest tests -m gpu -q -rs --durations=25 -p no:cacheprovider > gpurun_out/gputest_$T.txt 2>&1
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.txt 2>&1
bash tools/profile_round.sh $T
bash tools/workloads.sh $T > gpurun_out/workloads_$T.txt 2>&1
