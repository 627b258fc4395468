#!/bin/bash
# step stages of configs 4, 3, 5 with an environment switch at its values,
# interleaved over 3 repetitions: tools/ab_env_cfg.sh VAR v1 v2 ...
var=$1; shift
for rep in 1 2 3; do for c in 4 3 5; do for v in "$@"; do
  env $var=$v timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-solve --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d['stages_ms']
print('$var=$v cfg$c', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3), {k: round(v,3) for k,v in s.items()})"
done; done; done
