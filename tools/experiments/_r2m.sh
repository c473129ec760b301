O=gpurun_out/r02_n; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_allocator.py -q -x > $O/pytest_alloc.log 2>&1; echo "rc=$?" >> $O/pytest_alloc.log
tail -15 $O/pytest_alloc.log
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -4 $O/pytest_gpu.log
timeout 900 python bench.py --no-unscreened --no-cpu --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r02_n/bench.json").read().strip().splitlines()[-1])
print(d["ms_per_step"], d["roofline"]["frac"], d["roofline"]["kernel"], d["tune_s"])
print(d["granularity"])
print(" ".join(f'{c["cls"]}:{c["ms"]:.1f}:{c["variant"]}' for c in d["classes"][:14]))
PY
