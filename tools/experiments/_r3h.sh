# Strip layout sweep with dynamic strip hand-out (tools/strip_sweep.py).
O=gpurun_out/r03h; mkdir -p $O
timeout 1200 python tools/strip_sweep.py --waters 80 --set 1024,1024 --set 1024,256 --set 1024,512 --set 1024,2048 \
  --set 512,1024 --set 256,1024 --set 2048,1024 --set 1024,1024 > $O/sweep.txt 2>&1
cat $O/sweep.txt
