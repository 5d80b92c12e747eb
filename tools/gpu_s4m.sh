#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_cfg5_1gpu_r02_v9.json 2> gpurun_out/s4m.err; echo "cfg5 rc=$?"
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-graph > gpurun_out/s4m_cfg5_eager.json 2>> gpurun_out/s4m.err; echo "cfg5 eager rc=$?"
python tools/bsum.py gpurun_out/bench_cfg5_1gpu_r02_v9.json gpurun_out/s4m_cfg5_eager.json; tail -3 gpurun_out/s4m.err
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/s4m_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s4m_pytest.log; tail -3 gpurun_out/s4m_pytest.log
