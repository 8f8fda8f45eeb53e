# sweep of the one-warp thresholds (tools/var_b<BFS>e<ERO>.so), two passes, default workload then dem1000
for i in 1 2; do bash tools/variants.sh; done
for so in tools/var_*.so; do
  LEMGPU_LIB=$so timeout -s KILL 100 python bench.py --workload dem1000 --no-cpu-baseline --e2e-steps 0 --steps 50 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('dem1000 $so', round(d['ms_per_step'],4))"
done
