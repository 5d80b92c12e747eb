#!/bin/bash
# session-3 baseline: bench lines + full ncu captures with source of HEAD
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/s3a_cfg3.json 2> gpurun_out/s3a.err
timeout 300 python bench.py --config cfg2 --no-cpu-baseline --e2e-steps 1 > gpurun_out/s3a_cfg2.json 2>> gpurun_out/s3a.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"compact_kernel|sample_kernel" -s 2 -c 2 \
  -o gpurun_out/prof_s3a python tools/profile_scan.py --config cfg3 --trials 200000 --runs 2 > gpurun_out/ncu_s3a.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"primary_kernel" -s 1 -c 1 \
  -o gpurun_out/prof_s3a_primary python tools/profile_scan.py --config cfg2 --trials 100000 --runs 2 > gpurun_out/ncu_s3a_p.log 2>&1
tail -2 gpurun_out/ncu_s3a.log gpurun_out/ncu_s3a_p.log
head -c 400 gpurun_out/s3a_cfg3.json; echo; head -c 400 gpurun_out/s3a_cfg2.json
