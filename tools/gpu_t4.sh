cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --ignore=tests/test_gpu_full_size.py -rf > gpurun_out/t4_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t4_pytest.log
timeout 600 python tools/ab.py c5 LIB=abl/rows.so:rows base:mr --rounds 2 > gpurun_out/t4_ab_c5.jsonl 2>&1
timeout 900 python bench.py --gpus 4 --transport local --steps 3 > gpurun_out/t4_local4.json 2> gpurun_out/t4_local4.err
timeout 900 python bench.py --gpus 2 --transport local --steps 3 --workload c3 > gpurun_out/t4_local2_c3.json 2> gpurun_out/t4_local2_c3.err
