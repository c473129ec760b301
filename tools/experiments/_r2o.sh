O=gpurun_out/r02_o; mkdir -p $O
nproc > $O/nproc.txt; lscpu | grep "Model name" >> $O/nproc.txt
timeout 1200 python -m pytest tests/test_gpu_c5.py -q -x --durations=5 > $O/pytest_c5.log 2>&1; echo "rc=$?" >> $O/pytest_c5.log
tail -8 $O/pytest_c5.log
for n in 4 8; do
timeout 1200 python bench.py --geom ala$n --basis cc-pvtz --no-unscreened --no-cpu --steps 3 --warmup 3 > $O/bench_ala$n.json 2> $O/bench_ala$n.err
python - $O/bench_ala$n.json <<'PY'
import json, sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(d["config"]["workload"], d["config"]["n_basis"], d["ms_per_step"], d["roofline"]["frac"], d["roofline"].get("build_frac"), d["tune_s"])
print(" ".join(f'{c["cls"]}:{c["ms"]:.1f}:{c["variant"]}:{c["tflops"]:.1f}' for c in d["classes"][:16]))
PY
done
