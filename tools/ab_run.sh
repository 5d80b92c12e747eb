ARA_LIB_PATH=$PWD/gpurun_variants/r32.so timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash tools/ab_bench.sh cfg3 gpurun_variants/r64.so gpurun_variants/r32.so gpurun_variants/r64.so gpurun_variants/r32.so
