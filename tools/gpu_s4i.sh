#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for c in cfg1 cfg4; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/s4i_$c.json 2> gpurun_out/s4i_$c.err; echo "$c rc=$?"
  python tools/bsum.py gpurun_out/s4i_$c.json; tail -2 gpurun_out/s4i_$c.err
done
timeout 300 python bench.py --config cfg3 --plain-upload --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/s4i_plain.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/s4i_plain.json')); print('plain e2e', d['e2e']['value'])"
timeout 600 python bench.py --impl reference --config cfg2 --steps 2 --warmup 1 > gpurun_out/s4i_ref_cfg2.json 2>/dev/null; head -c 300 gpurun_out/s4i_ref_cfg2.json; echo
