#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
bash tools/build_variant.sh chk -DARA_DEVICE_CHECKS=1 > /dev/null 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/s3z_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s3z_pytest.log
tail -4 gpurun_out/s3z_pytest.log
ARA_LIB_PATH=$PWD/gpurun_variants/chk.so timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/r02_device_checks.log 2>&1; echo "pytest (ARA_DEVICE_CHECKS build) rc=$?" >> gpurun_out/r02_device_checks.log
tail -4 gpurun_out/r02_device_checks.log
