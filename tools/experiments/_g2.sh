O=gpurun_out/r02_ncu1; mkdir -p $O
timeout 900 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:Cls1000, 1, 1,|Cls0000, 1, 1,|jk_kernel<Cls1010" -c 3 -o $O/top \
  python tools/profile_build.py --waters 80 --builds 1 --set 1000=fam_x768 --set 0000=fam_pl768 --set 1010=lane_pl512 > $O/ncu_full.log 2>&1
echo "ncu rc=$?" >> $O/ncu_full.log
tail -3 $O/pytest_gpu.log; tail -3 $O/ncu_full.log
