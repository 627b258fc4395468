#!/bin/bash
# config-4 step and config-2 level-7 connectivity of library variants
# (lib/var_<name>; "base" = lib/): tools/ab_lib2.sh base x ...
for rep in 1 2; do for v in "$@"; do
  if [ "$v" = base ]; then lib=paper_2509_11133_b200/lib/libphfem.so; else lib=paper_2509_11133_b200/lib/var_$v/libphfem.so; fi
  PHFEM_LIB=$lib python bench.py --steps 10 --warmup 3 --no-solve --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d['stages_ms']
print('$v cfg4', round(d['ms_per_step'],3), {k: round(v,3) for k,v in s.items()})"
  PHFEM_LIB=$lib python bench.py --config 2 --steps 3 --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v cfg2', round(d['ms_per_step'],3), d['config']['levels'][-1]['connect_ms'])"
done; done
