#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for L in mz0 mz1 mz0 mz1; do ARA_LIB_PATH=$PWD/gpurun_variants/$L.so python tools/meas_async_timing.py | sed "s/^/$L /"; done > gpurun_out/s4r.log 2>&1
bash tools/ab_bench.sh cfg2 gpurun_variants/mz0.so gpurun_variants/mz1.so gpurun_variants/mz0.so gpurun_variants/mz1.so >> gpurun_out/s4r.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -k "measure or select or pml or tvar or var or exceed or sort or smoke" 2>&1 >> gpurun_out/s4r.log 2>&1; cat gpurun_out/s4r.log | tail -14
