set -x
python -m pytest tests -m gpu -q > gpurun_out/t_all_v22.log 2>&1; tail -3 gpurun_out/t_all_v22.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_v22.log 2>&1; tail -2 gpurun_out/smoke_v22.log
python bench.py > gpurun_out/bench_c2_v22.log 2>&1; tail -c 600 gpurun_out/bench_c2_v22.log
python bench.py --config 1 --steps 300 > gpurun_out/bench_c1_v22.log 2>&1
python bench.py --config 3 > gpurun_out/bench_c3_v22.log 2>&1
python bench.py --config 4 > gpurun_out/bench_c4_v22.log 2>&1
python bench.py --impl reference > gpurun_out/bench_ref_v22.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_v22.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_l_v22.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:multicrop_kernel -c 2 -f -o gpurun_out/mc_v22 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_v22.log 2>&1
ls -la gpurun_out | tail -5
