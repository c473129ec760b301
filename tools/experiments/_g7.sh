O=gpurun_out/r02_strip2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "strip or every_kernel" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
timeout 600 python bench.py --no-unscreened --no-cpu --steps 3 --warmup 2 > $O/bench.json 2> $O/bench.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r02_strip2/bench.json").read().strip().splitlines()[-1])
print(d["ms_per_step"], d["roofline"]["frac"], d["roofline"]["kernel"])
for c in d["classes"][:12]: print(c["cls"], c["ms"], c["variant"])
t=d["tune_ms"]
for k in ("1000","0000","1010","2010","1110","2000","1100"):
    print(k, {a:b for a,b in t.get(k,{}).items() if "strip" in a or a in ("fam_x768","fam_pl768","lane_pl512","lane_pl384","lane_sb512")})
PY
