timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash tools/ab_bench.sh cfg3 gpurun_variants/pre.so gpurun_variants/clip.so gpurun_variants/pre.so gpurun_variants/clip.so
