cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider --ignore=tests/test_gpu_full_size.py > gpurun_out/skip_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/skip_pytest.log
timeout 1500 python tools/ab.py c5 LIB=abl/base.so:base base:prod LIB=abl/skip.so,GGB_EXP_SKIP=8192:skip8k LIB=abl/skip.so,GGB_EXP_SKIP=16384:skip16k LIB=abl/skip.so,GGB_EXP_SKIP=28672:skip28k LIB=abl/skip.so,GGB_EXP_SKIP=65536:skip64k LIB=abl/skip.so,GGB_EXP_SKIP=262144:skip256k --rounds 2 > gpurun_out/ab_skip_c5.jsonl 2>&1
