#!/bin/bash
# config-4 step and config-2 level-7 connectivity with an environment
# switch at its values: tools/ab_env2.sh VAR v1 v2 ...
var=$1; shift
for rep in 1 2; do for v in "$@"; do
  env $var=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-solve --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d['stages_ms']
print('$var=$v cfg4', round(d['ms_per_step'],3), {k: round(v,3) for k,v in s.items()})"
  env $var=$v timeout 300 python bench.py --config 2 --steps 3 --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$var=$v cfg2', round(d['ms_per_step'],3), d['config']['levels'][-1]['connect_ms'])"
done; done
