# A/B of runtime knobs (env vars) by bench.py's step time and per-kernel CUDA-event sums
#   tools/gpu_ab_env.sh CONFIG "ENV1=a ENV2=b" "ENV1=c" ...
cfg=$1; shift
for E in "$@"; do
  env $E timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']['kernels']
print('$cfg [$E]', 'step_ms', round(d['ms_per_step'],3), 'trials/s %.4g' % d['value'], 'compact_sum', round(r['compact_kernel']['kernel_ms'],3), 'sample_sum', round(r['sample_kernel']['kernel_ms'],3), 'redo', round(r['redo_ms'],3), d['clocks']['sm_mhz'])"
done
