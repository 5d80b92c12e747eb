#!/bin/bash
# A/B the split kernels of several libara builds: per-kernel device time under ncu
# (serialised, cold cache: compare between builds, not to the bench).
#   tools/ab_kernels.sh lib1.so lib2.so ...
mkdir -p gpurun_out
for L in "$@"; do
  n=$(basename "$L" .so)
  ARA_LIB_PATH=$PWD/$L timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active \
     --clock-control none --csv --log-file gpurun_out/ab_$n.csv python tools/profile_scan.py --config ${AB_CONFIG:-cfg3} --trials 100000 --runs 1 > /dev/null 2>&1
  echo "== $n"; grep -E "compact|sample_kernel|scan_kernel" gpurun_out/ab_$n.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | sed 's/"//g' | head -8
done
