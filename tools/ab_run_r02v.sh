set -x
python -m pytest tests/test_gpu_store.py tests/test_loader_goldens.py -q -m gpu > gpurun_out/r02w_store_tests.log 2>&1; tail -n 2 gpurun_out/r02w_store_tests.log
bash tools/ab_c1.sh > gpurun_out/ab_c1d.log 2>&1
