#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x -rf -k "multirank" --durations=6 > gpurun_out/s4f_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s4f_pytest.log
tail -12 gpurun_out/s4f_pytest.log
bash tools/bench_multirank_check.sh cfg5 > gpurun_out/r02_v8_multirank_cfg5.log 2>&1; tail -2 gpurun_out/r02_v8_multirank_cfg5.log
