set -x
bash tools/ab_c1.sh > gpurun_out/ab_c1c.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:passthrough_kernel -s 3 -c 1 -f -o gpurun_out/pt_r02v python bench.py --config 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02v_ncu_pt.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02v_launches_c1.csv python bench.py --config 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02v_ncu_l1.log 2>&1
