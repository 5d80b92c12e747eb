#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
ARA_MEAS_CLUSTER_SIZE=8 timeout 120 python tools/meas_async_timing.py
ARA_MEAS_CLUSTER_SIZE=16 timeout 120 python tools/meas_async_timing.py
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"select_cluster" -s 3 -c 1 \
  -o gpurun_out/prof_s4d python tools/meas_async_timing.py > gpurun_out/ncu_s4d.log 2>&1
tail -1 gpurun_out/ncu_s4d.log
