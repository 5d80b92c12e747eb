timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
bash tools/ab_bench.sh cfg3 gpurun_variants/base2.so gpurun_variants/redux.so gpurun_variants/quint.so gpurun_variants/base2.so gpurun_variants/redux.so gpurun_variants/quint.so
