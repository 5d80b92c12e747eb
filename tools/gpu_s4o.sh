#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/s4o_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s4o_pytest.log; tail -3 gpurun_out/s4o_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_r02_v10.json 2> gpurun_out/bench_r02_v10.err
timeout 600 python bench.py --config cfg2 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg2_r02_v10.json 2>> gpurun_out/bench_r02_v10.err
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_cfg5_1gpu_r02_v10.json 2>> gpurun_out/bench_r02_v10.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r02_v10.json 2>> gpurun_out/bench_r02_v10.err
python tools/bsum.py gpurun_out/bench_r02_v10.json gpurun_out/bench_cfg2_r02_v10.json gpurun_out/bench_cfg5_1gpu_r02_v10.json
python -c "
import json
for f in ['gpurun_out/bench_r02_v10.json','gpurun_out/bench_cfg2_r02_v10.json','gpurun_out/bench_cfg5_1gpu_r02_v10.json']:
    d=json.load(open(f)); print(f, 'e2e', d['e2e']['value'], d['clocks'])
"
tail -2 gpurun_out/bench_r02_v10.err
