O=gpurun_out/r02_w; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_allocator.py -q -x -k "strip or granularity or tuned" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -2 $O/pytest.log
timeout 900 python bench.py --no-unscreened --no-cpu --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r02_w/bench.json").read().strip().splitlines()[-1])
print(d["ms_per_step"], d["roofline"]["frac"], d["roofline"]["kernel"], d["e2e"]["ms_per_step"])
print(" ".join(f'{c["cls"]}:{c["ms"]:.1f}:{c["variant"]}' for c in d["classes"][:12]))
PY
bash tools/ncu_traffic.sh 1000 fstrip_a_t512 | tail -12
