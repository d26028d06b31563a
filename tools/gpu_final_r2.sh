# Round-2 measurement set (one gpurun call, 1 GPU): bench lines c5 (+ e2e,
# cpu_baseline) and c1-c4, the reference CPU arm on c5, then the ncu
# evidence: launch list of the c5 bench command and a --set full capture of
# one c5 gg run's engine kernels (each ncu only after its command exited 0).
# The .ncu-rep stays in /tmp on the box (too large to bring back); its raw
# and source pages and the profiles/ summary come back as CSV / JSON.
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/f_smi.txt 2>&1
timeout 300 python -m pytest tests -m gpu -q -p no:cacheprovider --ignore=tests/test_gpu_full_size.py -rf -x > gpurun_out/f_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/f_pytest.log
timeout 420 python bench.py --steps 10 --warmup 3 > gpurun_out/f_bench_c5.json 2> gpurun_out/f_bench_c5.err
for w in c1 c2 c3 c4; do
  timeout 200 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/f_bench_$w.json 2> gpurun_out/f_bench_$w.err
done
timeout 500 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f_ref_c5.json 2> gpurun_out/f_ref_c5.err
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
  ncu -i /tmp/f_c5.ncu-rep --page raw --csv > gpurun_out/f_c5_raw.csv 2>/dev/null
  ncu -i /tmp/f_c5.ncu-rep --page details --csv -k regex:"edge_kernel<ggb::PageRank, void, 0>" -c 1 > gpurun_out/f_c5_dominant_details.csv 2>/dev/null
  ncu -i /tmp/f_c5.ncu-rep --page details --csv -k regex:edge_chain_kernel > gpurun_out/f_c5_chain_details.csv 2>/dev/null
  ncu -i /tmp/f_c5.ncu-rep --page source --csv --print-source cuda,sass -k regex:edge_chain_kernel > /tmp/f_chain_src.csv 2>/dev/null
  gzip -c /tmp/f_chain_src.csv > gpurun_out/f_c5_chain_source.csv.gz
  du -sh gpurun_out >> gpurun_out/f_ncu_full.log
fi
timeout 400 python bench.py --workload c5 --gpus 4 --transport local --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/f_bench_c5_local4.json 2> gpurun_out/f_bench_c5_local4.err
timeout 300 python bench.py --workload c4 --gpus 2 --transport local --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/f_bench_c4_local2.json 2> gpurun_out/f_bench_c4_local2.err
