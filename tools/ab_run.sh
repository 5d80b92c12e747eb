timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash tools/ab_bench.sh cfg3 gpurun_variants/c3.so gpurun_variants/c4.so gpurun_variants/c3.so gpurun_variants/c4.so
