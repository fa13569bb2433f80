#!/bin/bash
# Round-2 final measurement refresh on one B200 (run via gpurun); outputs land in gpurun_out/r02u_*
set -x
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02u_smoke.log 2>&1; tail -2 gpurun_out/r02u_smoke.log
python -m pytest tests -m gpu -q > gpurun_out/r02u_gpu_tests.log 2>&1; tail -2 gpurun_out/r02u_gpu_tests.log
python bench.py > gpurun_out/r02u_bench_c2.log 2>&1; tail -c 300 gpurun_out/r02u_bench_c2.log
python bench.py --config 1 --steps 300 > gpurun_out/r02u_bench_c1.log 2>&1
python bench.py --config 3 > gpurun_out/r02u_bench_c3.log 2>&1
python bench.py --config 4 > gpurun_out/r02u_bench_c4.log 2>&1
python bench.py --config 4 --tier-hbm-gb 40 --no-cpu-baseline > gpurun_out/r02u_bench_c4_tier40.log 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02u_bench_reference.log 2>&1
python tools/sampler_timing.py > gpurun_out/r02u_sampler_timing.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02u_launches_c2.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02u_ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:multicrop_kernel -c 2 -f -o gpurun_out/mc_r02u python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02u_ncu_mc.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"sample_(classify|eval|table|walk)" -s 4 -c 4 -f -o gpurun_out/smp_r02u python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02u_ncu_smp.log 2>&1
PF_SWEEP_DIR=gpurun_out python bench.py --config 5 > gpurun_out/r02u_sweep.log 2>&1; tail -c 200 gpurun_out/r02u_sweep.log
python tools/build_checks.py > /dev/null 2>&1 && PF_B200_LIB=$PWD/ab/checks.so python -m pytest tests -m gpu -q > gpurun_out/r02u_gpu_tests_pf_checks.log 2>&1; tail -2 gpurun_out/r02u_gpu_tests_pf_checks.log
ls -la gpurun_out | grep r02u | head -30
