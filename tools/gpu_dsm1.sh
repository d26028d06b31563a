cd $GRAFT_REPO_ROOT/tools
O=../gpurun_out/dsm1.txt
: > $O
for th in 256 512 1024; do timeout 120 ./dsmem_gather_bench ldg 1 13 5 $th >> $O 2>&1; done
for t in 12 13 14; do timeout 120 ./dsmem_gather_bench lds 1 $t 5 512 >> $O 2>&1; done
for c in 2 4 8 16; do for t in 12 13 14; do timeout 120 ./dsmem_gather_bench dsm $c $t 5 512 >> $O 2>&1; done; done
for c in 8 16; do timeout 120 ./dsmem_gather_bench dsm $c 13 5 1024 >> $O 2>&1; done
for c in 1 8 16; do for t in 13 14; do timeout 120 ./dsmem_gather_bench skip $c $t 5 512 >> $O 2>&1; done; done
cat $O
