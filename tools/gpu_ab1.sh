cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider --ignore=tests/test_gpu_full_size.py > gpurun_out/ab1_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab1_pytest.log
GGB_SMEM_HOT_KB=192 timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider --ignore=tests/test_gpu_full_size.py > gpurun_out/ab1_pytest_hot.log 2>&1; echo "rc=$?" >> gpurun_out/ab1_pytest_hot.log
timeout 1200 python tools/ab.py c5 LIB=abl/base.so:base base:new GGB_SMEM_HOT_KB=96:hot96 GGB_SMEM_HOT_KB=192:hot192 GGB_SMEM_HOT_KB=208:hot208 --rounds 2 > gpurun_out/ab1_c5.jsonl 2>&1
timeout 600 python tools/ab.py c4 LIB=abl/base.so:base base:new --rounds 2 > gpurun_out/ab1_c4.jsonl 2>&1
timeout 600 python tools/ab.py c3 LIB=abl/base.so:base base:new --rounds 2 > gpurun_out/ab1_c3.jsonl 2>&1
timeout 600 python tools/ab.py c2 LIB=abl/base.so:base base:new --rounds 2 > gpurun_out/ab1_c2.jsonl 2>&1
