O=gpurun_out/r02_l; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -30 $O/pytest.log | grep -v "^\s*$" | tail -12
timeout 600 python bench.py --no-unscreened --no-cpu --steps 3 --warmup 2 > $O/bench.json 2> $O/bench.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r02_l/bench.json").read().strip().splitlines()[-1])
print(d["ms_per_step"], d["roofline"]["frac"], d["roofline"]["kernel"])
for c in d["classes"][:12]: print(c["cls"], c["ms"], c["variant"])
t=d["tune_ms"]
for k in ("1000","0000","1010","2010","1110","2000","1100"):
    print(k, {a:b for a,b in sorted(t.get(k,{}).items(), key=lambda kv: kv[1])[:8]})
PY
