timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -6 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_cfg3.err
timeout 600 python bench.py --config cfg2 --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
python - <<'PY'
import json
for f in ("gpurun_out/bench_cfg3.json", "gpurun_out/bench_cfg2.json"):
    d = json.load(open(f)); r = d["roofline"]
    print(f, "%.4g trials/s" % d["value"], "%.3f ms" % d["ms_per_step"], {k: round(v["kernel_ms"], 3) for k, v in r["kernels"].items() if isinstance(v, dict)}, "e2e %.4g" % d["e2e"]["value"], "launches", d["gpu_launches"])
PY
