timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -12 gpurun_out/pytest_gpu.log
bash tools/gpu_ab_env.sh cfg3 "ARA_X=0" "ARA_SERIAL=1" "ARA_BATCH_TRIALS=8192" "ARA_BATCH_TRIALS=16384" "ARA_BATCH_TRIALS=65536" "ARA_BATCH_TRIALS=131072" "ARA_SERIAL=1 ARA_BATCH_TRIALS=800000"
bash tools/gpu_ab_env.sh cfg2 "ARA_X=0" "ARA_NO_PRIMARY_PATH=1"
