#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for c in cfg3 cfg2 cfg3; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 1 > gpurun_out/s3i_$c.json 2> gpurun_out/s3i.err
  python tools/bsum.py gpurun_out/s3i_$c.json
done
timeout 900 python -m pytest tests -m gpu -q -x -rf > gpurun_out/s3i_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s3i_pytest.log
tail -3 gpurun_out/s3i_pytest.log
