#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x -rf -k "large_catalog or measures_async" --durations=5 > gpurun_out/s3w_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s3w_pytest.log
tail -12 gpurun_out/s3w_pytest.log
