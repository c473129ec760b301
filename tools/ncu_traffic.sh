#!/bin/bash
# DRAM traffic of the dominant class launch ((ps|ss), unit kernels fam_x768:
# 4 member segments) for bench.py's roofline.traffic.
O=gpurun_out/r01traffic; mkdir -p $O
timeout 900 ncu --clock-control none --kernel-name-base demangled -k "regex:jk_fam_kernel<eritile_b200::Cls1000," -c 4 \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file $O/traffic.csv \
  python tools/profile_build.py --waters 80 --builds 1 --set 1000=fam_x768 > $O/log.txt 2>&1
tail -20 $O/traffic.csv
