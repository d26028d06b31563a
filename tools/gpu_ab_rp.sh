cd $GRAFT_REPO_ROOT
timeout 1500 python tools/ab.py c5 base:base LIB=abl/rp1.so:rp1 LIB=abl/rp2.so:rp2 --rounds 2 > gpurun_out/ab_rp_c5.jsonl 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/ab_rp_c5.jsonl'):
    d=json.loads(l)
    if 'error' in d: print(d['variant'], d['error'][-600:]); continue
    print(d['variant'], d['median_ms'], {k:(v['edge_ms'],v['rebuild_ms']) for k,v in d['modes'].items()})
PY
