O=gpurun_out/r02_k1; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -2 $O/pytest.log
timeout 1200 python bench.py --geom ala4 --basis cc-pvtz --no-unscreened --no-cpu --steps 3 --warmup 3 > $O/bench_ala4.json 2> $O/bench_ala4.err
timeout 900 python bench.py --no-unscreened --no-cpu --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err
python - <<'PY'
import json
for f in ("bench_ala4", "bench"):
    d=json.loads(open(f"gpurun_out/r02_k1/{f}.json").read().strip().splitlines()[-1])
    print(f, d["ms_per_step"], d["roofline"]["frac"], d["roofline"].get("build_frac"))
    print(" ".join(f'{c["cls"]}:{c["ms"]:.1f}:{c["variant"]}:{c["tflops"]:.1f}' for c in d["classes"][:16]))
PY
