# round-2 GPU check: all GPU parity tests (no -x: every failure listed), then the cfg3 / cfg2 bench lines
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -40 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --config cfg2 --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
tail -3 gpurun_out/bench.err
python - <<'PY'
import json
for f in ("gpurun_out/bench.json","gpurun_out/bench_cfg2.json"):
    try:
        d=json.load(open(f)); r=d["roofline"]["kernels"]
        print(f, d["value"], d["ms_per_step"], "compact", r["compact_kernel"]["kernel_ms"], "sample", r["sample_kernel"]["kernel_ms"], d["clocks"])
    except Exception as e: print(f, e)
PY
