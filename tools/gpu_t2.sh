cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --ignore=tests/test_gpu_full_size.py -rf > gpurun_out/t2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t2_pytest.log
timeout 1800 python -m pytest tests/test_gpu_full_size.py -s -q -p no:cacheprovider --durations=0 -rf > gpurun_out/t2_full.log 2>&1; echo "rc=$?" >> gpurun_out/t2_full.log
timeout 300 python tools/sanitize_case.py > gpurun_out/t2_sancase.log 2>&1; echo "rc=$?" >> gpurun_out/t2_sancase.log
