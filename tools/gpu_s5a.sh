#!/bin/bash
# run-to-run spread of the headline line: the default bench three times on one box
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for i in 1 2 3; do
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/rep_$i.json 2>/dev/null
  timeout 600 python bench.py --config cfg2 --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/rep2_$i.json 2>/dev/null
done
python - <<'PY' | tee gpurun_out/r02_v13_repeats.txt
import json
print("# tools/gpu_s5a.sh: bench.py three times on one box (cfg3 default steps; cfg2 30 steps)")
for cfg, pat in (("cfg3", "gpurun_out/rep_%d.json"), ("cfg2", "gpurun_out/rep2_%d.json")):
    for i in (1, 2, 3):
        d = json.load(open(pat % i))
        k = d["roofline"]["kernels"]
        print(cfg, i, "value %.4g trials/s" % d["value"], "ms/step %.4f" % d["ms_per_step"],
              "e2e %.4g" % d["e2e"]["value"], {n: round(v["kernel_ms"], 4) for n, v in k.items() if isinstance(v, dict)},
              "sm_mhz", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
