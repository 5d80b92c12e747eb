for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --steps 3 --e2e-steps 5 > gpurun_out/bp$i.json 2>/dev/null
timeout 600 python bench.py --no-cpu-baseline --steps 3 --e2e-steps 5 --plain-upload > gpurun_out/bu$i.json 2>/dev/null
done
python -c "
import json
for f in ('bp1','bu1','bp2','bu2'):
    d=json.load(open('gpurun_out/%s.json'%f)); print(f, d['e2e']['value'], d['e2e']['h2d_bytes_per_step'])"
nproc; lscpu | grep -i "numa node" | head -4
