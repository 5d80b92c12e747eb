#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x -rf > gpurun_out/s3t_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s3t_pytest.log
tail -5 gpurun_out/s3t_pytest.log
bash tools/ab_bench.sh cfg3 gpurun_variants/base8.so gpurun_variants/packx.so gpurun_variants/base8.so gpurun_variants/packx.so
