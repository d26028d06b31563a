cd $GRAFT_REPO_ROOT
timeout 60 python tools/dbg_small.py > gpurun_out/t13_dbg.log 2>&1; echo "rc=$?" >> gpurun_out/t13_dbg.log
timeout 400 python -m pytest tests -m gpu -q -p no:cacheprovider --ignore=tests/test_gpu_full_size.py -rf -x > gpurun_out/t13_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t13_pytest.log
timeout 500 python tools/ab.py c5 LIB=abl/head.so:head base:prod --rounds 2 > gpurun_out/t13_c5.jsonl 2>&1
timeout 300 python tools/ab.py c4 LIB=abl/head.so:head base:prod --rounds 1 > gpurun_out/t13_c4.jsonl 2>&1
timeout 200 python tools/ab.py c2 LIB=abl/head.so:head base:prod --rounds 2 > gpurun_out/t13_c2.jsonl 2>&1
