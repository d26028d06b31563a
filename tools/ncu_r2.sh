# round-2 ncu evidence for c5 (one gpurun call; ncu only after the same
# command exited 0 without it):
#  1. --set full of one gg run's engine kernels (first 14 matching launches:
#     initial sparsify/compaction + layout, 4 approximate gathers + epilogues,
#     the superstep chain + epilogue, the superstep rebuild compaction)
#  2. the launch list of the bench command (device time of every launch)
cd $GRAFT_REPO_ROOT
python tools/ncu_case.py --workload c5 --iters 7 > gpurun_out/r2_case_c5.txt 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"edge_kernel|edge_chain_kernel|vertex_kernel|scan_compact|sp_layout" -c 14 \
    -o gpurun_out/r2_c5 -f python tools/ncu_case.py --workload c5 --iters 7 > gpurun_out/r2_ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/r2_ncu_full.log
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_plain.json 2> gpurun_out/r2_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c5_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_ncu_launch.log 2>&1
echo "launch rc=$?" >> gpurun_out/r2_ncu_launch.log
