#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for c in cfg3 cfg2 cfg1; do
  for fl in "" "--no-graph"; do
    timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 $fl > gpurun_out/s4k_$c$fl.json 2> gpurun_out/s4k.err; echo "$c $fl rc=$?"
    python tools/bsum.py gpurun_out/s4k_$c$fl.json
  done
done
tail -3 gpurun_out/s4k.err
timeout 1200 python -m pytest tests -m gpu -q -x -rf -k "multirank" > gpurun_out/s4k_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s4k_pytest.log; tail -3 gpurun_out/s4k_pytest.log
timeout 600 python bench.py > gpurun_out/s4k_default.json 2>/dev/null; python tools/bsum.py gpurun_out/s4k_default.json; python -c "
import json; d=json.load(open('gpurun_out/s4k_default.json')); print(d['config']['launch'], d['gpu_launches'], d['cpu_baseline']['value'], d['e2e']['value'])"
