cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --ignore=tests/test_gpu_full_size.py -rf > gpurun_out/t5_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t5_pytest.log
timeout 2000 python -m pytest tests/test_gpu_full_size.py -s -q -rf -p no:cacheprovider --durations=0 > gpurun_out/t5_full.log 2>&1; echo "rc=$?" >> gpurun_out/t5_full.log
