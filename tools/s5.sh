timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "host or dropin or cpp" -p no:cacheprovider 2>&1 | tail -2
timeout -s KILL 600 python -m pytest tests/test_lem_cli.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
timeout -s KILL 300 python tools/e2e_prof.py 10000 2>&1 | tail -4
timeout -s KILL 400 python bench.py --steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step'], d['e2e']['frac_of_copy_floor'])"
