# Strip kernels with fewer, fatter threads (384 / 256 threads, up to 168 / 255 registers).
O=gpurun_out/r03d; mkdir -p $O
timeout 900 python tools/variant_compare.py --waters 80 > $O/compare.txt 2>&1
cat $O/compare.txt
