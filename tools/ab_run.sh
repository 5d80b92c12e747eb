timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b3.json 2>gpurun_out/b3.err; tail -2 gpurun_out/b3.err
timeout 600 python bench.py --no-cpu-baseline --plain-upload > gpurun_out/b3p.json 2>/dev/null
python -c "
import json
for f in ('gpurun_out/b3.json','gpurun_out/b3p.json'):
    d=json.load(open(f)); print(f, d['ms_per_step'], d['value'], d['e2e'])"
