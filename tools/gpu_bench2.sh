cd $GRAFT_REPO_ROOT
timeout 900 python bench.py > gpurun_out/b2_c5.json 2> gpurun_out/b2_c5.err
timeout 900 python bench.py --gpus 4 --transport local --steps 3 > gpurun_out/b2_local4.json 2> gpurun_out/b2_local4.err
timeout 900 python bench.py --gpus 2 --transport local --steps 3 --workload c4 > gpurun_out/b2_local2_c4.json 2> gpurun_out/b2_local2_c4.err
