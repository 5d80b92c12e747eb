#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for c in cfg2 cfg3 cfg2 cfg3; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 1 > gpurun_out/s3v_$c.json 2>> gpurun_out/s3v.err
  python tools/bsum.py gpurun_out/s3v_$c.json
done
tail -3 gpurun_out/s3v.err
