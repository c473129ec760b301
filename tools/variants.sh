timeout 300 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for v in libvar_m2_p600.so libvar_m2_p0.so libvar_m3_p600.so libvar_m3_p0.so; do
  ERITILE_LIBNAME=$v python bench.py --no-cpu --steps 3 --warmup 2 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],1), ' '.join(c['cls']+':'+str(round(c['ms'],1)) for c in d['classes'][:7]))"
done
