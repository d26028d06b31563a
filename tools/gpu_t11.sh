cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --ignore=tests/test_gpu_full_size.py -rf > gpurun_out/t11_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t11_pytest.log
timeout 1200 python tools/ab.py c5 LIB=abl/base.so:base base:prod --rounds 2 > gpurun_out/t11_c5.jsonl 2>&1
timeout 900 python tools/ab.py c2 LIB=abl/base.so:base base:prod --rounds 2 > gpurun_out/t11_c2.jsonl 2>&1
timeout 2000 python -m pytest tests/test_gpu_full_size.py -s -q -rf -p no:cacheprovider > gpurun_out/t11_full.log 2>&1; echo "rc=$?" >> gpurun_out/t11_full.log
