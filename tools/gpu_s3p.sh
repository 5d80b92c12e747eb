#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -rf > gpurun_out/s3p_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s3p_pytest.log
tail -3 gpurun_out/s3p_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3p_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s3p_smoke.log; tail -2 gpurun_out/s3p_smoke.log
bash tools/capture_profiles.sh r02_v5
python tools/bsum.py gpurun_out/bench_r02_v5.json gpurun_out/bench_cfg2_r02_v5.json gpurun_out/bench_cfg5_1gpu_r02_v5.json
bash tools/bench_multirank_check.sh cfg3 > gpurun_out/r02_v5_multirank_cfg3.log 2>&1; tail -3 gpurun_out/r02_v5_multirank_cfg3.log
bash tools/bench_multirank_check.sh cfg5 > gpurun_out/r02_v5_multirank_cfg5.log 2>&1; tail -3 gpurun_out/r02_v5_multirank_cfg5.log
