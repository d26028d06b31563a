cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests -m gpu -q -p no:cacheprovider --ignore=tests/test_gpu_full_size.py -rf -x > gpurun_out/t12_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t12_pytest.log
timeout 500 python tools/ab.py c5 LIB=abl/base.so:base base:prod --rounds 2 > gpurun_out/t12_c5.jsonl 2>&1
timeout 300 python tools/ab.py c2 LIB=abl/base.so:base base:prod --rounds 2 > gpurun_out/t12_c2.jsonl 2>&1
timeout 600 python -m pytest tests/test_gpu_full_size.py -s -q -rf -x -p no:cacheprovider > gpurun_out/t12_full.log 2>&1; echo "rc=$?" >> gpurun_out/t12_full.log
