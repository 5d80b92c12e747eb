#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -rf > gpurun_out/s3m_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s3m_pytest.log
tail -3 gpurun_out/s3m_pytest.log
for c in cfg2 cfg3 cfg2 cfg3; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 1 > gpurun_out/s3m_$c.json 2>> gpurun_out/s3m.err
  python tools/bsum.py gpurun_out/s3m_$c.json
done
timeout 300 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/s3m_cfg5.json 2>> gpurun_out/s3m.err
python tools/bsum.py gpurun_out/s3m_cfg5.json
for gb in 67108864 268435456; do ARA_GROUP_BYTES=$gb timeout 300 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/s3m_cfg5_$gb.json 2>> gpurun_out/s3m.err; python tools/bsum.py gpurun_out/s3m_cfg5_$gb.json; done
