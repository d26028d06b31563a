cd $GRAFT_REPO_ROOT
timeout 1500 python tools/ab.py c5 LIB=abl/base.so:base base:prod LIB=abl/skip.so,GGB_EXP_SKIP=0:skip0 LIB=abl/skip.so,GGB_EXP_SKIP=8192:skip8k LIB=abl/skip.so,GGB_EXP_SKIP=28672:skip28k LIB=abl/skip.so,GGB_EXP_SKIP=262144:skip256k LIB=abl/skip.so,GGB_EXP_SKIP=2097152:skip2m --rounds 2 > gpurun_out/ab_skip2_c5.jsonl 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:edge_chain_kernel -c 1 -o gpurun_out/chain_c5 -f python tools/ncu_case.py --workload c5 --iters 5 > gpurun_out/ncu_chain.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_chain.log
