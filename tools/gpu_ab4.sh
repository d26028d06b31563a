cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider --ignore=tests/test_gpu_full_size.py > gpurun_out/ab4_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab4_pytest.log
timeout 1200 python tools/ab.py c5 LIB=abl/base.so:base base:prod LIB=abl/nofilt.so:claimonly --rounds 2 > gpurun_out/ab4_c5.jsonl 2>&1
timeout 900 python tools/ab.py c2 LIB=abl/base.so:base base:prod --rounds 2 > gpurun_out/ab4_c2.jsonl 2>&1
timeout 900 python tools/ab.py c4 LIB=abl/base.so:base base:prod --rounds 1 > gpurun_out/ab4_c4.jsonl 2>&1
