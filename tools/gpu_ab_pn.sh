cd $GRAFT_REPO_ROOT
GGB_LIB_PATH=$GRAFT_REPO_ROOT/abl/pn.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pagerank or chain_stress or hub_windows or random_graphs or grid_and_thread or tile_boundaries or exactness or ties or invalid" > gpurun_out/pn_tests.log 2>&1; tail -3 gpurun_out/pn_tests.log
timeout 1500 python tools/ab.py c5 base:base LIB=abl/pn.so:pn --rounds 3 > gpurun_out/ab_pn_c5.jsonl 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/ab_pn_c5.jsonl'):
    d=json.loads(l)
    if 'error' in d: print(d['variant'], d['error'][-600:]); continue
    print(d['variant'], d['median_ms'], {k:(v['edge_ms'],v['rebuild_ms']) for k,v in d['modes'].items()})
PY
