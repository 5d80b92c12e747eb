#!/bin/bash
# A/B libara variants on cfg2 (primary path): tools/ab_cfg2.sh lib1.so lib2.so ...
for L in "$@"; do
  ARA_LIB_PATH=$PWD/$L timeout 300 python bench.py --config cfg2 --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']['kernels']
print('$L', round(d['ms_per_step'],4), 'primary', round(r['primary_kernel']['kernel_ms'],4), 'meas', round(r['gather_and_measures_ms'],4))"
done
