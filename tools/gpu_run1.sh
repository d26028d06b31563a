cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider --ignore=tests/test_gpu_full_size.py > gpurun_out/pytest_main.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_main.log
timeout 1500 python -m pytest tests/test_gpu_full_size.py -s -q -rf -p no:cacheprovider --durations=0 > gpurun_out/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
