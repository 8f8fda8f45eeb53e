# runtime pipeline knobs on 10000^2: bands x tile CTAs per band
for i in 1 2; do
for o in '{}' '{"pipe": 20}' '{"pipe": 28}' '{"pipe_tile_grid": 518}' '{"pipe_tile_grid": 666}' '{"pipe_tile_grid": 560}' '{"pipe_tile_grid": 620}'; do
  timeout -s KILL 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --options "$o" 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('dem10000 $o', round(d['ms_per_step'],4))"
done; done
