for L in liblemgpu_orig liblemgpu liblemgpu_s64 liblemgpu_s256 liblemgpu_orig; do
  LEMGPU_LIB=paper_1803_02977_b200/$L.so python bench.py --steps 20 --e2e-steps 0 --no-cpu-baseline | python -c "import json,sys; d=json.load(sys.stdin); print('$L', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms']['k_tiles'],4))"
done
./oracle/_ref/test_dropin 2>&1 | tail -15
