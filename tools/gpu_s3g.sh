#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests -m gpu -q -x -rf -k "measures" > gpurun_out/s3g_pytest_meas.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s3g_pytest_meas.log
tail -3 gpurun_out/s3g_pytest_meas.log
timeout 120 python tools/meas_async_timing.py; ARA_MEAS_TAIL=0 timeout 120 python tools/meas_async_timing.py
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"select_tail" -s 8 -c 3 \
  -o gpurun_out/prof_s3g_tail python tools/meas_async_timing.py > gpurun_out/ncu_s3g.log 2>&1
tail -1 gpurun_out/ncu_s3g.log
