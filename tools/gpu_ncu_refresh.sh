# Refresh the ncu evidence of the c5 step after a kernel change: launch list of
# the bench command and a --set full capture of one gg run's engine kernels
# (each ncu only after its command exited 0 without it).
cd $GRAFT_REPO_ROOT
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f_plain.json 2> gpurun_out/f_plain.err && \
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_c5_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f_ncu_launch.log 2>&1
echo "launch rc=$?" >> gpurun_out/f_ncu_launch.log
timeout 200 python tools/ncu_case.py --workload c5 --iters 7 > gpurun_out/f_case_c5.txt 2>&1 && \
timeout 700 ncu --set full --clock-control none --import-source on \
    -k regex:"edge_kernel|edge_chain_kernel|vertex_kernel|scan_compact|sp_layout" -c 14 \
    -o /tmp/f_c5 -f python tools/ncu_case.py --workload c5 --iters 7 > gpurun_out/f_ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/f_ncu_full.log
if [ -f /tmp/f_c5.ncu-rep ]; then
  python tools/ncu_summary2.py /tmp/f_c5.ncu-rep c5 gpurun_out/f_case_c5.txt >> gpurun_out/f_ncu_full.log 2>&1
  cp profiles/ncu_c5.json gpurun_out/f_ncu_c5.json
  ncu -i /tmp/f_c5.ncu-rep --page details --csv -k regex:"edge_kernel<ggb::PageRank, void, 0>" -c 1 > gpurun_out/f_c5_dominant_details.csv 2>/dev/null
fi
tail -3 gpurun_out/f_ncu_launch.log gpurun_out/f_ncu_full.log
