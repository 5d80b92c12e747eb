#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/s3d_cfg3.json 2> gpurun_out/s3d.err
python tools/bsum.py gpurun_out/s3d_cfg3.json
timeout 900 python -m pytest tests -m gpu -q -x -rf > gpurun_out/s3d_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s3d_pytest.log
tail -4 gpurun_out/s3d_pytest.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"compact_kernel|sample_kernel" -s 2 -c 2 \
  -o gpurun_out/prof_s3d python tools/profile_scan.py --config cfg3 --trials 200000 --runs 2 > gpurun_out/ncu_s3d.log 2>&1
tail -1 gpurun_out/ncu_s3d.log
