cd $GRAFT_REPO_ROOT
ncu --set full --clock-control none --import-source on -k regex:"edge_chain_kernel" -c 1 -o gpurun_out/r2_chain4_c5 -f python tools/ncu_case.py --workload c5 --iters 5 > gpurun_out/r2_chain_ncu.log 2>&1; tail -2 gpurun_out/r2_chain_ncu.log
