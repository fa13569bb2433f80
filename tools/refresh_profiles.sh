#!/bin/bash
# Round-2 measurement refresh on one B200 (run via gpurun); outputs land in gpurun_out/r02f_*
set -x
python bench.py > gpurun_out/r02f_bench_c2.log 2>&1; tail -c 300 gpurun_out/r02f_bench_c2.log
python bench.py --config 1 --steps 300 > gpurun_out/r02f_bench_c1.log 2>&1
python bench.py --config 3 > gpurun_out/r02f_bench_c3.log 2>&1
python bench.py --config 4 > gpurun_out/r02f_bench_c4.log 2>&1
python bench.py --config 4 --tier-hbm-gb 40 --no-cpu-baseline > gpurun_out/r02f_bench_c4_tier40.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02f_launches_c2.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02f_ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:multicrop_kernel -c 2 -f -o gpurun_out/mc_r02 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02f_ncu_mc.log 2>&1
ls -la gpurun_out | grep r02f | head -20
