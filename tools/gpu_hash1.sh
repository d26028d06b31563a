cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sparsify or tile_boundaries or presparsified or c1_pagerank or random_graphs" > gpurun_out/hash_tests.log 2>&1; tail -3 gpurun_out/hash_tests.log
timeout 900 python tools/ab.py c5 base:newhash --rounds 2 > gpurun_out/ab_hash_c5.jsonl 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/ab_hash_c5.jsonl'):
    d=json.loads(l); print(d.get('variant'), d.get('median_ms'), d.get('error','')[-300:])
PY
