# Dynamic, heaviest-first strip hand-out: per-class times, full GPU suite, headline bench.
O=gpurun_out/r03e; mkdir -p $O
timeout 900 python tools/variant_compare.py --waters 80 > $O/compare.txt 2>&1
cat $O/compare.txt
timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -2 $O/pytest_gpu.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
python -c "import json; d=json.load(open('$O/bench.json')); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['frac'], d['clocks'])"
