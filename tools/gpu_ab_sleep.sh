cd $GRAFT_REPO_ROOT
timeout 1500 python tools/ab.py c5 base:base LIB=abl/sl0.so:sl0 LIB=abl/sl20.so:sl20 LIB=abl/sl200.so:sl200 --rounds 2 > gpurun_out/ab_sleep_c5.jsonl 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/ab_sleep_c5.jsonl'):
    d=json.loads(l)
    if 'error' in d: print(d['variant'], d['error'][-600:]); continue
    print(d['variant'], d['median_ms'], {k:(v['edge_ms'],v['rebuild_ms']) for k,v in d['modes'].items()})
PY
