# Warp-specialised strip variants (OPT 256): parity of every strip variant, then
# per-class times against the round-2 choices on (H2O)_80.
O=gpurun_out/r03b; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k strip > $O/pytest_strip.log 2>&1; echo "rc=$?" >> $O/pytest_strip.log
tail -3 $O/pytest_strip.log
timeout 900 python tools/variant_compare.py --waters 80 > $O/compare.txt 2>&1
timeout 600 python tools/variant_compare.py --waters 80 --cls 1000,1010,0000 --var strip_o7_t512,strip_a_t512,strip_w_t768,strip_wa_t768 >> $O/compare.txt 2>&1
cat $O/compare.txt
