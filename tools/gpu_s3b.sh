#!/bin/bash
# build, full GPU test suite, bench lines cfg3/cfg2/cfg5
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/s3b_cfg3.json 2> gpurun_out/s3b.err
timeout 300 python bench.py --config cfg2 --no-cpu-baseline --e2e-steps 1 > gpurun_out/s3b_cfg2.json 2>> gpurun_out/s3b.err
timeout 1500 python -m pytest tests -m gpu -q -x -rf --durations=15 > gpurun_out/s3b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s3b_pytest.log
tail -25 gpurun_out/s3b_pytest.log
timeout 300 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/s3b_cfg5.json 2>> gpurun_out/s3b.err
tail -3 gpurun_out/s3b.err
