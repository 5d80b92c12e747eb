#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -rf -k "measures" > gpurun_out/s4c_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s4c_pytest.log
tail -8 gpurun_out/s4c_pytest.log
timeout 120 python tools/meas_async_timing.py; ARA_MEAS_CLUSTER=0 timeout 120 python tools/meas_async_timing.py
for i in 1 2; do timeout 300 python bench.py --config cfg2 --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/s4c_cfg2.json 2>/dev/null; python tools/bsum.py gpurun_out/s4c_cfg2.json; done
for i in 1 2; do ARA_MEAS_CLUSTER=0 timeout 300 python bench.py --config cfg2 --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/s4c_cfg2.json 2>/dev/null; python tools/bsum.py gpurun_out/s4c_cfg2.json; done
