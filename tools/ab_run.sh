bash tools/ab_bench.sh cfg3 gpurun_variants/s96.so gpurun_variants/s64.so gpurun_variants/s80.so gpurun_variants/s128.so gpurun_variants/s96.so gpurun_variants/s64.so gpurun_variants/s80.so
