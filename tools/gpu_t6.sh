cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --ignore=tests/test_gpu_full_size.py -rf > gpurun_out/t6_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t6_pytest.log
timeout 1200 python tools/ab.py c5 LIB=abl/base.so:base base:split --rounds 2 > gpurun_out/t6_c5.jsonl 2>&1
timeout 900 python tools/ab.py c2 LIB=abl/base.so:base base:split --rounds 2 > gpurun_out/t6_c2.jsonl 2>&1
timeout 900 python tools/ab.py c4 LIB=abl/base.so:base base:split --rounds 1 > gpurun_out/t6_c4.jsonl 2>&1
timeout 900 python tools/ab.py c3 LIB=abl/base.so:base base:split --rounds 1 > gpurun_out/t6_c3.jsonl 2>&1
