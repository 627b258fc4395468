#!/bin/bash
# config-4 step stages of library variants (lib/var_<name>; "base" = lib/),
# interleaved over 3 repetitions: tools/ab_cfg4.sh base x ...
for rep in 1 2 3; do for v in "$@"; do
  if [ "$v" = base ]; then lib=paper_2509_11133_b200/lib/libphfem.so; else lib=paper_2509_11133_b200/lib/var_$v/libphfem.so; fi
  PHFEM_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-solve --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d['stages_ms']
print('$v cfg4', round(d['ms_per_step'],3), d.get('roofline',{}).get('kernel_ms'), {k: round(v,3) for k,v in s.items()})"
done; done
