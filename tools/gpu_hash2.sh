cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sparsify or tile_boundaries or presparsified" > gpurun_out/hash_tests.log 2>&1; tail -2 gpurun_out/hash_tests.log
timeout 900 python tools/ab.py c5 base:newhash3 --rounds 2 > gpurun_out/ab_hash3_c5.jsonl 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/ab_hash3_c5.jsonl'):
    d=json.loads(l); print(d.get('variant'), d.get('median_ms'), d.get('error','')[-300:])
PY
ncu --set full --clock-control none --import-source on -k regex:"scan_compact" -c 1 -o gpurun_out/r2_scan3_c5 -f python tools/ncu_case.py --workload c5 --iters 2 > gpurun_out/r2_scan_ncu.log 2>&1; tail -2 gpurun_out/r2_scan_ncu.log
