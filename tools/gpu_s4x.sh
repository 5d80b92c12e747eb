#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/r02_v13_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_v13_pytest_gpu.log
tail -3 gpurun_out/r02_v13_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_r02_v13.json 2> gpurun_out/bench_r02_v13.err; echo "bench rc=$?"
timeout 600 python bench.py --config cfg2 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg2_r02_v13.json 2>> gpurun_out/bench_r02_v13.err
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_cfg5_1gpu_r02_v13.json 2>> gpurun_out/bench_r02_v13.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r02_v13.json 2>> gpurun_out/bench_r02_v13.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_v13.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_under_ncu_r02_v13.log 2>&1
python tools/bsum.py gpurun_out/bench_r02_v13.json gpurun_out/bench_cfg2_r02_v13.json gpurun_out/bench_cfg5_1gpu_r02_v13.json
