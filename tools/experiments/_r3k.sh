# Strip layout (tools/strip_layout.py), each layout tuned.
O=gpurun_out/r03k; mkdir -p $O
timeout 1800 python tools/strip_layout.py --waters 80 --set 1024,1024 --set 1024,4096 --set 256,1024 --set 256,4096 --set 4096,1024 > $O/layout.txt 2>&1
cat $O/layout.txt
