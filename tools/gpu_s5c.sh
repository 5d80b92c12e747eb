#!/bin/bash
# per-rank proxy of the 8-GPU sharded cfg3 run: cfg3's shape at 100k trials on one GPU
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 600 python bench.py --config configs/cfg3_100k_rank_share.json --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/cfg3_100k.json 2> gpurun_out/cfg3_100k.err
timeout 600 python bench.py --config configs/cfg3_100k_rank_share.json --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --no-graph > gpurun_out/cfg3_100k_nograph.json 2>> gpurun_out/cfg3_100k.err
python tools/bsum.py gpurun_out/cfg3_100k.json gpurun_out/cfg3_100k_nograph.json
tail -2 gpurun_out/cfg3_100k.err
