#!/bin/bash
# The bench's multi-rank path (trial shards, YLT all-gather, measures on the
# gathered [P][L][N/P] layout, max-over-ranks timing) on ONE GPU: 2 ranks
# share it over gloo.  The measures must equal the 1-rank run's.
set -e
cfg=${1:-cfg1}
timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/mr_1.json
ARA_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29533 bench.py --config $cfg --gpus 2 --steps 3 --warmup 3 \
    --no-cpu-baseline --e2e-steps 1 > gpurun_out/mr_2.json 2> gpurun_out/mr_2.err || (tail -20 gpurun_out/mr_2.err; exit 1)
python - <<'PY'
import json
a = json.load(open("gpurun_out/mr_1.json")); b = json.loads(open("gpurun_out/mr_2.json").read().strip().splitlines()[-1])
print("1 rank:", a["value"], a["measures"]); print("2 ranks:", b["n_gpus"], b["value"], b["measures"], b["config"]["parallelism"])
assert a["measures"] == b["measures"], "measures differ between 1 and 2 ranks"
print("multi-rank measures identical")
PY
