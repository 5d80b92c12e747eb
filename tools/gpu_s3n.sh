#!/bin/bash
mkdir -p gpurun_out
for L in head_ec6 bulk head_ec6 bulk; do
  ARA_LIB_PATH=$PWD/gpurun_variants/$L.so timeout 300 python bench.py --config cfg2 --steps 20 --no-cpu-baseline --e2e-steps 1 > gpurun_out/s3n_$L.json 2>> gpurun_out/s3n.err
  echo $L; python tools/bsum.py gpurun_out/s3n_$L.json
done
ARA_LIB_PATH=$PWD/gpurun_variants/bulk.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3n_launches.csv python bench.py --config cfg2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/s3n_launches.csv | head -12
