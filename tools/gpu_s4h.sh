#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x -rf -k "vs_oracle_sort" --durations=4 > gpurun_out/s4h_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s4h_pytest.log
tail -8 gpurun_out/s4h_pytest.log
