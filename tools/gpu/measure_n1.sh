#!/bin/bash
# round-2 measurements at HEAD: bench N=1 (driver settings), ncu launch list of the
# same command (cold, serialised: shares only), one ncu --set full capture of the climb kernel
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_n1.json 2> gpurun_out/r02_bench_n1.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2> gpurun_out/r02_ncu_launch.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_hill_async -c 1 -o gpurun_out/r02_c3_full python tools/run_search.py C3 full 1 > gpurun_out/r02_ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_default -s 1 -c 1 -o gpurun_out/r02_c3_default python tools/run_search.py C3 default 1 > gpurun_out/r02_ncu_default.log 2>&1
