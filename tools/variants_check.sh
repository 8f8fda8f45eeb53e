#!/bin/bash
# Quick parity (1000^2 anchors + schedule cross-checks) and the default bench per tools/var_*.so.
for so in tools/var_*.so; do
  r=$(LEMGPU_LIB=$so timeout -s KILL 200 python -m pytest tests/test_gpu_parity.py -x -q -k "anchor_1000 or schedules_agree" 2>&1 | tail -1)
  echo "$so: $r"
done
bash tools/variants.sh
