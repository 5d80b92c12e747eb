# ncu capture of the current split kernels (cfg3, 200k trials) + the 2-ranks-on-1-GPU bench check
tag=${1:-r02_v2}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"compact_kernel|sample_kernel" -s 2 -c 2 \
  -o gpurun_out/prof_${tag} python tools/profile_scan.py --config cfg3 --trials 200000 --runs 2 > gpurun_out/ncu_${tag}.log 2>&1
tail -1 gpurun_out/ncu_${tag}.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"primary_kernel" -s 1 -c 1 \
  -o gpurun_out/prof_${tag}_primary python tools/profile_scan.py --config cfg2 --trials 100000 --runs 2 > gpurun_out/ncu_${tag}_p.log 2>&1
tail -1 gpurun_out/ncu_${tag}_p.log
bash tools/bench_multirank_check.sh cfg1 > gpurun_out/multirank_cfg1.log 2>&1; tail -3 gpurun_out/multirank_cfg1.log
bash tools/bench_multirank_check.sh cfg3 > gpurun_out/multirank_cfg3.log 2>&1; tail -3 gpurun_out/multirank_cfg3.log
