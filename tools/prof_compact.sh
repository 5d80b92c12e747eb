# ncu --set full of one compact_kernel launch (cfg3, 200k trials) -> gpurun_out/$1.ncu-rep
timeout 600 ncu --set full --import-source on --clock-control none -k regex:${2:-compact_kernel} -s 1 -c 1 -o gpurun_out/$1 python tools/profile_scan.py --config ${3:-cfg3} --trials 200000 --runs 2 > gpurun_out/ncu_$1.log 2>&1; tail -2 gpurun_out/ncu_$1.log
