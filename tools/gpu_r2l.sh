timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -6 gpurun_out/pytest_gpu.log
for c in cfg3 cfg2; do
timeout 600 python bench.py --config $c --no-cpu-baseline --e2e-steps 2 > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err; python -c "
import json; d=json.load(open('gpurun_out/b_$c.json')); k=d['roofline']['kernels']
print('$c', round(d['ms_per_step'],4), '%.4g trials/s' % d['value'], {a: (round(b['kernel_ms'],3) if isinstance(b, dict) else round(b,4)) for a,b in k.items()}, 'e2e %.4g' % d['e2e']['value'], d['gpu_launches'])" || tail -3 gpurun_out/b_$c.err
done
