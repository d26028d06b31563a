cd $GRAFT_REPO_ROOT/tools
O=../gpurun_out/dsm2.txt
: > $O
for th in 256 512; do
for md in ldg pol1 pol2; do timeout 120 ./dsmem_gather_bench $md 1 13 10 $th >> $O 2>&1; done
for t in 14 15; do timeout 120 ./dsmem_gather_bench win 1 $t 10 $th >> $O 2>&1; done
done
cat $O
