# ncu of the sampler for several libara builds (cfg3, 200k trials)
for L in "$@"; do
  n=$(basename $L .so)
  ARA_LIB_PATH=$PWD/$L timeout 600 ncu --set full --clock-control none -k regex:"sample_kernel" -s 1 -c 1 \
    -o gpurun_out/ab_$n python tools/profile_scan.py --config cfg3 --trials 200000 --runs 2 > gpurun_out/ab_$n.log 2>&1
  tail -1 gpurun_out/ab_$n.log
done
