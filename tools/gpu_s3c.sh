#!/bin/bash
mkdir -p gpurun_out
for pb in 0 4096 8192 16384 32768 65536; do ARA_MEAS_PER_BLOCK=$pb timeout 120 python tools/meas_async_timing.py; done > gpurun_out/s3c_meas.txt 2>&1
cat gpurun_out/s3c_meas.txt
for L in gpurun_variants/base3.so gpurun_variants/pf1.so gpurun_variants/base3.so gpurun_variants/pf1.so; do
  ARA_LIB_PATH=$PWD/$L timeout 300 python bench.py --config cfg2 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/s3c_cfg2_$(basename $L .so).json 2>/dev/null
  python tools/bsum.py gpurun_out/s3c_cfg2_$(basename $L .so).json
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"primary_kernel" -s 1 -c 1 \
  -o gpurun_out/prof_s3c_primary python tools/profile_scan.py --config cfg2 --trials 100000 --runs 2 > gpurun_out/ncu_s3c_p.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"select_multi" -s 3 -c 2 \
  -o gpurun_out/prof_s3c_meas python tools/meas_async_timing.py > gpurun_out/ncu_s3c_m.log 2>&1
tail -1 gpurun_out/ncu_s3c_p.log gpurun_out/ncu_s3c_m.log
