#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 600 python bench.py > gpurun_out/s4q_cfg3.json 2> gpurun_out/s4q.err; echo "cfg3 rc=$?"
timeout 600 python bench.py --config cfg2 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/s4q_cfg2.json 2>> gpurun_out/s4q.err; echo "cfg2 rc=$?"
python tools/bsum.py gpurun_out/s4q_cfg3.json gpurun_out/s4q_cfg2.json
python -c "
import json
for f in ['gpurun_out/s4q_cfg3.json','gpurun_out/s4q_cfg2.json']:
    d=json.load(open(f)); print(f, 'e2e', d['e2e']['value'], d['e2e'].get('plain_uint32',{}).get('value'))"
timeout 900 python -m pytest tests -m gpu -q -k "multirank or smoke or e2e" 2>&1 | tail -2
tail -3 gpurun_out/s4q.err
