#!/bin/bash
# Time one config/algo under several env settings: variants_cfg.sh CFG ALGO RECORDS "ENV=.." ...
cfg=$1; algo=$2; recs=$3; shift 3
zs=${ZIPF_S:-0}
for v in "$@"; do
  env $v timeout 300 python tools/prof_run.py --config $cfg --algo $algo --records $recs --zipf-s $zs > gpurun_out/var.log 2>&1
  python - "$v" <<'PY'
import json, sys
t = open('gpurun_out/var.log').read()
try:
    d = json.loads(t[t.index('{'):])
    print(sys.argv[1], {k: round(v[1], 3) for k, v in d['kernels'].items() if v[1] > 0.05},
          {k: d['metrics'][k] for k in ('grace_levels', 'child_subpasses', 'recursion_depth')})
except Exception as e:
    print(sys.argv[1], 'FAILED', t[-300:])
PY
done
