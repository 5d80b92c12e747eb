ARA_LIB_PATH=$PWD/gpurun_variants/l1.so timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
bash tools/ab_bench.sh cfg3 gpurun_variants/l0.so gpurun_variants/l1.so gpurun_variants/l0.so gpurun_variants/l1.so
