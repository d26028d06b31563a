cd $GRAFT_REPO_ROOT
timeout 1500 python tools/ab.py c5 base:hot24 GGB_HOT_KB=12288:hot12 GGB_HOT_KB=16384:hot16 GGB_HOT_KB=32768:hot32 GGB_HOT_KB=49152:hot48 --rounds 2 > gpurun_out/ab_hot_c5.jsonl 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/ab_hot_c5.jsonl'):
    d=json.loads(l)
    if 'error' in d: print(d['variant'], d['error'][-600:]); continue
    print(d['variant'], d['median_ms'], {k:(v['edge_ms'],v['rebuild_ms']) for k,v in d['modes'].items()})
PY
