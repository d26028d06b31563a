cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --ignore=tests/test_gpu_full_size.py -rf > gpurun_out/t3_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t3_pytest.log
bash tools/ncu_r2.sh
