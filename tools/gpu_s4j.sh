#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for c in cfg1 cfg2 cfg3; do timeout 300 python tools/graph_timing.py $c 30 2>&1 | tail -3; done
