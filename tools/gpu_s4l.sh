#!/bin/bash
# round-2 end bench lines (graph-replayed steps) + launch list
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python bench.py > gpurun_out/bench_r02_v9.json 2> gpurun_out/bench_r02_v9.err
timeout 600 python bench.py --config cfg2 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg2_r02_v9.json 2>> gpurun_out/bench_r02_v9.err
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_cfg5_1gpu_r02_v9.json 2>> gpurun_out/bench_r02_v9.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r02_v9.json 2>> gpurun_out/bench_r02_v9.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_v9.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_under_ncu_r02_v9.log 2>&1
python tools/bsum.py gpurun_out/bench_r02_v9.json gpurun_out/bench_cfg2_r02_v9.json gpurun_out/bench_cfg5_1gpu_r02_v9.json
head -c 300 gpurun_out/bench_ref_r02_v9.json; echo
tail -2 gpurun_out/bench_r02_v9.err
