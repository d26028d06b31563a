cd $GRAFT_REPO_ROOT
GGB_LIB_PATH=$GRAFT_REPO_ROOT/abl/int.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -m gpu -x -q > gpurun_out/int_tests.log 2>&1; tail -3 gpurun_out/int_tests.log
timeout 1500 python tools/ab.py c5 base:base LIB=abl/int.so:interior --rounds 3 > gpurun_out/ab_int_c5.jsonl 2>&1
timeout 600 python tools/ab.py c2 base:base LIB=abl/int.so:interior --rounds 2 > gpurun_out/ab_int_c2.jsonl 2>&1
python - <<'PY'
import json
for f in ('c5','c2'):
  for l in open(f'gpurun_out/ab_int_{f}.jsonl'):
    d=json.loads(l)
    if 'error' in d: print(d['variant'], d['error'][-600:]); continue
    print(f, d['variant'], d['median_ms'], {k:(v['edge_ms'],v['rebuild_ms']) for k,v in d['modes'].items()})
PY
