for rep in 1 2; do for h in 0 1; do PHFEM_GROUPS_HASH=$h python bench.py --steps 10 --warmup 3 --no-solve --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d['stages_ms']
print('hash=$h', round(d['ms_per_step'],3), {k: round(v,3) for k,v in s.items()})"; done; done
