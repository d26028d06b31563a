cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --ignore=tests/test_gpu_full_size.py -rf > gpurun_out/t10_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t10_pytest.log
timeout 900 python bench.py --gpus 4 --transport local --steps 3 --workload c4 > gpurun_out/t10_local4_c4.json 2> gpurun_out/t10_local4_c4.err
timeout 900 python bench.py --gpus 4 --transport local --steps 3 --workload c4 --no-fused > gpurun_out/t10_local4_c4_nf.json 2> gpurun_out/t10_local4_c4_nf.err
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/t10_bench_c5.json 2> gpurun_out/t10_bench_c5.err
