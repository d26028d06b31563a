cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider --ignore=tests/test_gpu_full_size.py > gpurun_out/x1_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/x1_pytest.log
timeout 1200 python tools/ab.py c5 LIB=abl/base.so:base base:rows --rounds 2 > gpurun_out/x1_c5.jsonl 2>&1
timeout 600 python tools/ab.py c4 LIB=abl/base.so:base base:rows --rounds 2 > gpurun_out/x1_c4.jsonl 2>&1
timeout 600 python tools/ab.py c3 LIB=abl/base.so:base base:rows --rounds 2 > gpurun_out/x1_c3.jsonl 2>&1
timeout 600 python tools/ab.py c2 LIB=abl/base.so:base base:rows --rounds 2 > gpurun_out/x1_c2.jsonl 2>&1
timeout 600 python tools/ab.py c1 LIB=abl/base.so:base base:rows --rounds 2 > gpurun_out/x1_c1.jsonl 2>&1
timeout 1500 python -m pytest tests/test_gpu_full_size.py -s -q -x -p no:cacheprovider > gpurun_out/x1_full.log 2>&1; echo "rc=$?" >> gpurun_out/x1_full.log
