for i in 1 2; do bash tools/variants.sh; done
for so in tools/var_*.so; do LEMGPU_LIB=$so timeout -s KILL 200 python bench.py --workload ens64 --steps 10 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('ens64 $so', round(d['ms_per_step'],4))"; done
