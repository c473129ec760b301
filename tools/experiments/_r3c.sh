# Warp-specialised strip variants after the pre-claim fix: strip parity (every
# strip variant), per-class times incl. the 1024-thread half split.
O=gpurun_out/r03c; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k strip > $O/pytest_strip.log 2>&1; echo "rc=$?" >> $O/pytest_strip.log
tail -3 $O/pytest_strip.log
timeout 900 python tools/variant_compare.py --waters 80 > $O/compare.txt 2>&1
cat $O/compare.txt
