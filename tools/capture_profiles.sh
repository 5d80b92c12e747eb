#!/bin/bash
# Round-end evidence (one GPU): full ncu captures of the split kernels (cfg3's
# first 200k trials) and of the primary kernel (cfg2's first 100k trials), the
# launch list of a short bench run, and the bench lines (cfg3, cfg2, cfg5 on one
# GPU, the oracle reference arm).
#   tools/capture_profiles.sh TAG
tag=${1:-r02}
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"compact_kernel|sample_kernel" -s 2 -c 2 \
  -o gpurun_out/prof_${tag} python tools/profile_scan.py --config cfg3 --trials 200000 --runs 2 > gpurun_out/ncu_${tag}.log 2>&1
tail -1 gpurun_out/ncu_${tag}.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"primary_kernel" -s 1 -c 1 \
  -o gpurun_out/prof_${tag}_primary python tools/profile_scan.py --config cfg2 --trials 100000 --runs 2 > gpurun_out/ncu_${tag}_p.log 2>&1
tail -1 gpurun_out/ncu_${tag}_p.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${tag}.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_under_ncu_${tag}.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err
timeout 600 python bench.py --config cfg2 --no-cpu-baseline > gpurun_out/bench_cfg2_${tag}.json 2>> gpurun_out/bench_${tag}.err
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_cfg5_1gpu_${tag}.json 2>> gpurun_out/bench_${tag}.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_${tag}.json 2>> gpurun_out/bench_${tag}.err
cat gpurun_out/bench_${tag}.json | head -c 600; echo
