#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/r02_v12_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_v12_pytest_gpu.log
tail -3 gpurun_out/r02_v12_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_r02_v12.json 2> gpurun_out/bench_r02_v12.err; echo "bench rc=$?"
python tools/bsum.py gpurun_out/bench_r02_v12.json
