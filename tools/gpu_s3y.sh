#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
bash tools/build_variant.sh chk -DARA_DEVICE_CHECKS=1 > /dev/null 2>&1
echo "== normal build"; timeout 600 python -m pytest tests -m gpu -q -x -k "large_catalog" 2>&1 | tail -3
echo "== chk build"; ARA_LIB_PATH=$PWD/gpurun_variants/chk.so timeout 600 python -m pytest tests -m gpu -q -x -k "large_catalog" 2>&1 | tail -3
echo "== chk build, blocking"; CUDA_LAUNCH_BLOCKING=1 ARA_LIB_PATH=$PWD/gpurun_variants/chk.so timeout 600 python -m pytest tests -m gpu -q -x -k "large_catalog and False" 2>&1 | grep -E "Error|error|passed|failed" | head -10
echo "== normal build, both orders"; timeout 600 python -m pytest tests -m gpu -q -x -k "large_catalog and False" 2>&1 | tail -2
