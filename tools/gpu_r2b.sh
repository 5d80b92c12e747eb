# round 2: parity tests + bench + a full ncu capture of both split kernels (cfg3, 200k trials)
tag=${1:-r02}
timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
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
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"compact_kernel|sample_kernel" -s 2 -c 2 \
  -o gpurun_out/prof_${tag} python tools/profile_scan.py --config cfg3 --trials 200000 --runs 2 > gpurun_out/ncu_${tag}.log 2>&1
tail -2 gpurun_out/ncu_${tag}.log
