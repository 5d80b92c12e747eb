#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for L in m4 m3 m4 m3; do ARA_LIB_PATH=$PWD/gpurun_variants/$L.so timeout 300 python tools/meas_async_timing.py | sed "s/^/$L /"; done > gpurun_out/s4s.log 2>&1
bash tools/ab_bench.sh cfg2 gpurun_variants/m4.so gpurun_variants/m3.so gpurun_variants/m4.so gpurun_variants/m3.so >> gpurun_out/s4s.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x >> gpurun_out/s4s.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s4s.log
cat gpurun_out/s4s.log | grep -v "^\.\.\." | tail -16
