# 640-thread strip variants: per-class times, then the tuned bench.
O=gpurun_out/r03m; mkdir -p $O
timeout 900 python tools/variant_compare.py --waters 80 > $O/compare.txt 2>&1
cat $O/compare.txt
timeout 1200 python bench.py --no-unscreened > $O/bench.json 2> $O/bench.err
python -c "import json; d=json.load(open('$O/bench.json')); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel']); print({c['cls']: c['variant'] for c in d['classes'][:8]})"
