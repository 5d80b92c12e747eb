timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -8 gpurun_out/pytest_gpu.log
bash tools/ab_bench.sh cfg3 paper_1310_2274_b200/lib/libara.so gpurun_variants/ftz_c.so paper_1310_2274_b200/lib/libara.so gpurun_variants/ftz_c.so
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/cfg5.json 2> gpurun_out/cfg5.err
python -c "
import json; d=json.load(open('gpurun_out/cfg5.json')); r=d['roofline']['kernels']
print('cfg5 1 GPU', round(d['ms_per_step'],3), 'ms', '%.4g trials/s' % d['value'], 'compact', round(r['compact_kernel']['kernel_ms'],3), 'sample', round(r['sample_kernel']['kernel_ms'],3), d['portfolio'])" || tail -3 gpurun_out/cfg5.err
