timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
bash tools/ab_bench.sh cfg3 paper_1310_2274_b200/lib/libara.so gpurun_variants/v1.so gpurun_variants/v2slow.so paper_1310_2274_b200/lib/libara.so gpurun_variants/v1.so
bash tools/gpu_ab_env.sh cfg3 "ARA_BATCH_TRIALS=800000" "ARA_BATCH_TRIALS=131072" "ARA_BATCH_TRIALS=65536"
bash tools/gpu_ab_env.sh cfg2 "ARA_X=0"
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_full.err
