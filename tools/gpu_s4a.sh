#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
bash tools/ab_bench.sh cfg3 gpurun_variants/base9.so gpurun_variants/modes.so gpurun_variants/base9.so gpurun_variants/modes.so
timeout 1200 python -m pytest tests -m gpu -q -x -rf -k "exact or capped or redo or table_less or sampler or degenerate or async" > gpurun_out/s4a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s4a_pytest.log
tail -3 gpurun_out/s4a_pytest.log
