cd $GRAFT_REPO_ROOT/tools
for sh in 0.1 0.2 0.3 0.4; do timeout 120 ./tma_gather_bench mix 0 5 $sh; done > ../gpurun_out/tma2.txt 2>&1
timeout 120 ./tma_gather_bench ldg 0 5 >> ../gpurun_out/tma2.txt 2>&1
