timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python tools/meas_timing.py
ARA_MEASURES_SORT=1 python tools/meas_timing.py
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/b3.json 2>/dev/null
timeout 600 python bench.py --config cfg2 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b2.json 2>/dev/null
python -c "
import json
for f in ('gpurun_out/b3.json','gpurun_out/b2.json'):
    d=json.load(open(f)); print(f, d['ms_per_step'], d['roofline']['path_hbm']['run_ms'], d['value'])"
