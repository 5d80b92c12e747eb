timeout 600 python -m pytest tests -m gpu -q -x -rf -k "group_byte or large_portfolio or cfg5" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
for B in 68719476736 134217728 67108864; do
  ARA_GROUP_BYTES=$B timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/cfg5_$B.json 2> gpurun_out/cfg5_$B.err
  python -c "
import json; d=json.load(open('gpurun_out/cfg5_$B.json')); r=d['roofline']['kernels']
print('ARA_GROUP_BYTES=$B', round(d['ms_per_step'],3), 'ms', '%.4g trials/s' % d['value'], 'compact', round(r['compact_kernel']['kernel_ms'],3), 'sample', round(r['sample_kernel']['kernel_ms'],3), 'launches', d['gpu_launches'])" || tail -3 gpurun_out/cfg5_$B.err
done
