#!/bin/bash
# A/B libara variants by bench.py's per-kernel CUDA-event times
#   tools/ab_bench.sh CONFIG lib1.so lib2.so ...
cfg=$1; shift
for L in "$@"; do
  ARA_LIB_PATH=$PWD/$L timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']['kernels']
print('$L', round(d['ms_per_step'],4), ' '.join(f'{k} {round(v[\"kernel_ms\"],4)}' for k, v in r.items() if isinstance(v, dict)), d['clocks']['sm_mhz'])"
done
