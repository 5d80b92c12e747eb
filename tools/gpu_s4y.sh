#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
bash tools/ab_bench.sh cfg2 gpurun_variants/p2.so gpurun_variants/p3.so gpurun_variants/p2.so gpurun_variants/p3.so
