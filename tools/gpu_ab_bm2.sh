cd $GRAFT_REPO_ROOT
GGB_LIB_PATH=$GRAFT_REPO_ROOT/abl/bm2.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -m gpu -x -q > gpurun_out/bm2_tests.log 2>&1; tail -3 gpurun_out/bm2_tests.log
for w in c2 c3 c4; do timeout 600 python tools/ab.py $w base:base LIB=abl/bm2.so:bmask2 --rounds 2 > gpurun_out/ab_bm2_$w.jsonl 2>&1; done
python - <<'PY'
import json
for w in ('c2','c3','c4'):
  for l in open(f'gpurun_out/ab_bm2_{w}.jsonl'):
    d=json.loads(l)
    if 'error' in d: print(w, d['variant'], d['error'][-600:]); continue
    print(w, d['variant'], d['median_ms'], {k:(v['edge_ms'],v['rebuild_ms']) for k,v in d['modes'].items()})
PY
