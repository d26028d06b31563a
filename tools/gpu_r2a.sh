cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rf -p no:cacheprovider --ignore=tests/test_gpu_full_size.py --durations=15 > gpurun_out/a_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/a_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/a_bench_c5.json 2> gpurun_out/a_bench_c5.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/a_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/a_smoke.log
