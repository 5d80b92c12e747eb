#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/s4t_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s4t_pytest.log
tail -3 gpurun_out/s4t_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash tools/capture_profiles.sh r02_v11
python tools/bsum.py gpurun_out/bench_r02_v11.json gpurun_out/bench_cfg2_r02_v11.json gpurun_out/bench_cfg5_1gpu_r02_v11.json
timeout 300 python bench.py --config cfg2 --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_cfg2_30_r02_v11.json 2>/dev/null
python tools/bsum.py gpurun_out/bench_cfg2_30_r02_v11.json
