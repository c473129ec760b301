O=gpurun_out/r02_d; mkdir -p $O
for L in liberitile_b200.so liberitile_b200_mixed.so; do
ERITILE_LIBNAME=$L timeout 600 python bench.py --no-unscreened --no-cpu --steps 3 --warmup 2 > $O/bench_$L.json 2> $O/bench_$L.err
echo "== $L"
python - $O/bench_$L.json <<'PY'
import json, sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(d["ms_per_step"], d["roofline"]["frac"], d["roofline"]["kernel"])
print(" ".join(f'{c["cls"]}:{c["ms"]:.1f}:{c["variant"]}' for c in d["classes"][:14]))
t=d["tune_ms"]
for k in ("1000","0000","1010","2010","1110","2000","1100"):
    print(k, {a:b for a,b in sorted(t.get(k,{}).items(), key=lambda kv: kv[1])[:6]})
PY
done
