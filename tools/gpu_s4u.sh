#!/bin/bash
# the GPU suite against a bounds-checked build (ARA_DEVICE_CHECKS: __trap on a failed check), final build
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
ARA_LIB_PATH=$PWD/gpurun_variants/chk.so timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/r02_device_checks_final.log 2>&1; echo "pytest (ARA_DEVICE_CHECKS build) rc=$?" >> gpurun_out/r02_device_checks_final.log
tail -4 gpurun_out/r02_device_checks_final.log
