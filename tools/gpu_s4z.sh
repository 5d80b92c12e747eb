#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for L in g2 g3 g2 g3; do ARA_LIB_PATH=$PWD/gpurun_variants/$L.so timeout 300 python tools/meas_async_timing.py | sed "s/^/$L /"; done > gpurun_out/s4z.log 2>&1
bash tools/ab_bench.sh cfg2 gpurun_variants/g2.so gpurun_variants/g3.so gpurun_variants/g2.so gpurun_variants/g3.so >> gpurun_out/s4z.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -k "measures or adversarial or smoke or multirank or oep or exceed" >> gpurun_out/s4z.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s4z.log
grep -v "^\.\.\." gpurun_out/s4z.log | tail -14
