timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
bash tools/ab_bench.sh cfg3 gpurun_variants/store_ord.so gpurun_variants/ftz_c.so gpurun_variants/store_ord.so gpurun_variants/ftz_c.so
bash tools/ab_bench.sh cfg5 gpurun_variants/store_ord.so
