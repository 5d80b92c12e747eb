#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/s4e_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s4e_pytest.log
tail -3 gpurun_out/s4e_pytest.log
timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/s4e_cfg3.json 2>/dev/null; python tools/bsum.py gpurun_out/s4e_cfg3.json
