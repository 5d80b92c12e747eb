#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -rf -k "packed or supplied_z_survives or async" > gpurun_out/s4n_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s4n_pytest.log; tail -3 gpurun_out/s4n_pytest.log
for c in cfg3 cfg2; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 8 > gpurun_out/s4n_$c.json 2> gpurun_out/s4n.err; echo "$c rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/s4n_$c.json')); e=d['e2e']; print('$c', round(d['value']/1e6,1), 'e2e', round(e['value']/1e6,2), 'plain', round(e['plain_uint32']['value']/1e6,2))"
done
tail -3 gpurun_out/s4n.err
