O=gpurun_out/r02_v; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_c5.py tests/test_gpu_parity.py -q -x  > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
timeout 1200 python bench.py --geom ala4 --basis cc-pvtz --no-unscreened --no-cpu --steps 3 --warmup 3 > $O/bench_ala4.json 2> $O/bench_ala4.err
python - $O/bench_ala4.json <<'PY'
import json, sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(d["config"]["n_basis"], d["ms_per_step"], d["roofline"]["frac"], d["roofline"].get("build_frac"), d["tune_s"])
print(" ".join(f'{c["cls"]}:{c["ms"]:.1f}:{c["variant"]}:{c["tflops"]:.1f}' for c in d["classes"][:16]))
PY
