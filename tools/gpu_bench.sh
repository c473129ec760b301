#!/bin/bash
# Quick bench-only GPU call: bench JSON to gpurun_out/<tag>/bench.json
TAG=${1:-quick}; shift
O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python bench.py --no-cpu --no-unscreened "$@" > $O/bench.json 2> $O/bench.err
python - "$O/bench.json" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("ms/build", round(d["ms_per_step"], 2), "quartets/s %.3e" % d["value"], "tune_s", round(d.get("tune_s", 0), 1))
for c in d["classes"][:14]:
    t = d.get("tune_ms", {}).get(c["cls"], {})
    print(c["cls"], c["variant"], round(c["ms"], 1), round(c["tflops"], 2), " ".join(f"{k}={v:.1f}" for k, v in t.items()))
PY
