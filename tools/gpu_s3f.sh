#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests -m gpu -q -x -rf -k "measures" > gpurun_out/s3f_pytest_meas.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s3f_pytest_meas.log
tail -15 gpurun_out/s3f_pytest_meas.log
for pb in 0; do timeout 120 python tools/meas_async_timing.py; ARA_MEAS_TAIL=0 timeout 120 python tools/meas_async_timing.py; done
for c in cfg2 cfg3; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 1 > gpurun_out/s3f_$c.json 2> gpurun_out/s3f.err
  python tools/bsum.py gpurun_out/s3f_$c.json
done
timeout 300 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/s3f_cfg5.json 2>> gpurun_out/s3f.err
python tools/bsum.py gpurun_out/s3f_cfg5.json
