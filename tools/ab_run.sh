timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash tools/ab_bench.sh cfg3 gpurun_variants/rb0.so gpurun_variants/rb1.so gpurun_variants/rb0.so gpurun_variants/rb1.so
for L in rb0 rb1; do ARA_LIB_PATH=$PWD/gpurun_variants/$L.so timeout 600 python bench.py --config cfg5 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']['kernels']
print('cfg5 $L', round(d['ms_per_step'],3), 'compact', round(r['compact_kernel']['kernel_ms'],3), 'sample', round(r['sample_kernel']['kernel_ms'],3))"; done
