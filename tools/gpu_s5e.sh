#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
bash tools/ab_bench.sh cfg3 gpurun_variants/base.so gpurun_variants/c24.so gpurun_variants/c28.so gpurun_variants/base.so gpurun_variants/c24.so gpurun_variants/c28.so
