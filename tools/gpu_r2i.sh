timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
# memcheck over the round-2 kernels: overflow pass, primary path, supplied draws, batching, groups, fp64 solver
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests -m gpu -q -x \
  -k "overflow or primary or supplied or batching or group_byte or fp64_solver or heavy_overlap or rng_modes_vs_oracle or occ_max_redo" \
  > gpurun_out/r02_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/r02_memcheck.log
tail -5 gpurun_out/r02_memcheck.log
