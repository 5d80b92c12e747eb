#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for v in 1 0 1 0; do
  ARA_COMPACT_IX4=$v timeout 300 python bench.py --config cfg3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/s3j_ix$v.json 2> gpurun_out/s3j.err
  python tools/bsum.py gpurun_out/s3j_ix$v.json
done
timeout 900 python -m pytest tests -m gpu -q -x -rf > gpurun_out/s3j_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s3j_pytest.log
tail -3 gpurun_out/s3j_pytest.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"compact_kernel" -s 1 -c 1 \
  -o gpurun_out/prof_s3j python tools/profile_scan.py --config cfg3 --trials 200000 --runs 2 > gpurun_out/ncu_s3j.log 2>&1
tail -1 gpurun_out/ncu_s3j.log
