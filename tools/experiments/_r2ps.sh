O=gpurun_out/r02_ps; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -2 $O/pytest.log
timeout 900 python bench.py --no-unscreened --no-cpu --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r02_ps/bench.json").read().strip().splitlines()[-1])
print(d["ms_per_step"], d["roofline"]["frac"], d["roofline"]["kernel"])
print(" ".join(f'{c["cls"]}:{c["ms"]:.1f}:{c["variant"]}' for c in d["classes"][:12]))
t=d["tune_ms"]
for k in ("1000","0000","1010","1100","2000","2100","1110"):
    print(k, {a:b for a,b in sorted(t.get(k,{}).items(), key=lambda kv: kv[1]) if a.startswith("lane_p")})
PY
