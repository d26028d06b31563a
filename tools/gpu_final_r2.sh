# Round-2 measurement set (one gpurun call, 1 GPU): bench lines c5 (+ e2e,
# cpu_baseline) and c1-c4, the reference CPU arm on c5, then the ncu
# evidence: launch list of the c5 bench command and a --set full capture of
# one c5 gg run's engine kernels (each ncu only after its command exited 0).
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/f_smi.txt 2>&1
timeout 420 python bench.py --steps 10 --warmup 3 > gpurun_out/f_bench_c5.json 2> gpurun_out/f_bench_c5.err
for w in c1 c2 c3 c4; do
  timeout 240 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/f_bench_$w.json 2> gpurun_out/f_bench_$w.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f_ref_c5.json 2> gpurun_out/f_ref_c5.err
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f_plain.json 2> gpurun_out/f_plain.err && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_c5_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f_ncu_launch.log 2>&1
echo "launch rc=$?" >> gpurun_out/f_ncu_launch.log
timeout 300 python tools/ncu_case.py --workload c5 --iters 7 > gpurun_out/f_case_c5.txt 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"edge_kernel|edge_chain_kernel|vertex_kernel|scan_compact|sp_layout" -c 14 \
    -o gpurun_out/f_c5 -f python tools/ncu_case.py --workload c5 --iters 7 > gpurun_out/f_ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/f_ncu_full.log
