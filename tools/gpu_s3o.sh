#!/bin/bash
# sanitizers over the session-3 kernel changes: bulk bitmap copies (mbarrier), VEC / packed-index
# compaction, flat primary pipeline, constant degenerate tables, async measures
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
SEL="not full_size and not cfg5_rank_shard and not every_sort_size and not many_return_periods and not vs_oracle_sort"
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests -m gpu -q -x -k "$SEL" \
  > gpurun_out/r02_s3_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/r02_s3_memcheck.log
tail -4 gpurun_out/r02_s3_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests -m gpu -q -x \
  -k "primary or integer or sharding or heavy or async" > gpurun_out/r02_s3_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/r02_s3_racecheck.log
tail -4 gpurun_out/r02_s3_racecheck.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests -m gpu -q -x \
  -k "primary or integer or sharding or heavy" > gpurun_out/r02_s3_synccheck.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/r02_s3_synccheck.log
tail -4 gpurun_out/r02_s3_synccheck.log
