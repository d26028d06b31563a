cd $GRAFT_REPO_ROOT
timeout 1200 python tools/ab.py c5 LIB=abl/base.so:base base:prod LIB=abl/ldz.so:ldz LIB=abl/lb7.so:lb7 --rounds 2 > gpurun_out/ab3_c5.jsonl 2>&1
timeout 900 python tools/ab.py c4 LIB=abl/base.so:base base:prod LIB=abl/ldz.so:ldz --rounds 2 > gpurun_out/ab3_c4.jsonl 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:edge_chain_kernel -c 1 -o gpurun_out/chain_c5 -f python tools/ncu_case.py --workload c5 --iters 5 > gpurun_out/ncu_chain.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_chain.log
