bash tools/ab_bench.sh cfg3 gpurun_variants/cg0.so gpurun_variants/cg1.so gpurun_variants/cg2.so gpurun_variants/cg0.so gpurun_variants/cg1.so gpurun_variants/cg2.so
