for i in 1 2; do for so in tools/var_base.so tools/var_pf.so; do
  LEMGPU_LIB=$so timeout -s KILL 100 python bench.py --no-cpu-baseline --e2e-steps 0 --steps 30 "$@" 2>/dev/null \
    | python -c "import json,sys; d=json.load(sys.stdin); k=d['roofline']['kernel_ms']; print('$so', round(d['ms_per_step'],4), {a: round(b,4) for a,b in k.items()})"
done; done
