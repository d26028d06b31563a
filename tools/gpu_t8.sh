cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --ignore=tests/test_gpu_full_size.py -rf > gpurun_out/t8_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t8_pytest.log
timeout 1200 python tools/ab.py c5 LIB=abl/base.so:base base:prod --rounds 2 > gpurun_out/t8_c5.jsonl 2>&1
timeout 900 python tools/ab.py c2 LIB=abl/base.so:base base:prod --rounds 2 > gpurun_out/t8_c2.jsonl 2>&1
timeout 900 python tools/ab.py c4 LIB=abl/base.so:base base:prod --rounds 1 > gpurun_out/t8_c4.jsonl 2>&1
timeout 600 python tools/rows_c5.py c5 > gpurun_out/t8_rows_c5.json 2>&1
