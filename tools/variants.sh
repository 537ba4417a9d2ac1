#!/bin/bash
# Time C2 under several env settings (one prof_run per setting); prints kernel ms.
for v in "$@"; do
  env $v timeout 200 python tools/prof_run.py --config C2 > gpurun_out/var.log 2>&1
  python - "$v" <<'PY'
import json, sys
t = open('gpurun_out/var.log').read()
try:
    d = json.loads(t[t.index('{'):])
    print(sys.argv[1], {k: round(v[1], 3) for k, v in d['kernels'].items() if v[1] > 0.05})
except Exception as e:
    print(sys.argv[1], 'FAILED', t[-300:])
PY
done
