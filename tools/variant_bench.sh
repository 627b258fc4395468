#!/bin/bash
# Interleaved cfg4 bench of experiment builds: tools/variant_bench.sh name... (lib/var_<name>; "base" = lib/)
# prints ms/step and the assembly-kernel / stage times per run
for rep in 1 2; do
  for v in "$@"; do
    if [ "$v" = base ]; then lib=paper_2509_11133_b200/lib/libphfem.so; else lib=paper_2509_11133_b200/lib/var_$v/libphfem.so; fi
    PHFEM_LIB=$lib python bench.py --steps 10 --warmup 3 --no-solve --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d['stages_ms']
print('$v', round(d['ms_per_step'],3), 'asmk', round(s['assemble_kernel'],3), 'groups', round(s['groups'],3), 'number', round(s['number'],3), 'star', round(s['star'],3))"
  done
done
