O=gpurun_out/r02_f; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:jk_strip_kernel<eritile_b200::Cls1000, \(bool\)1, \(int\)1, \(int\)1|jk_strip_kernel<eritile_b200::Cls0000, \(bool\)1, \(int\)1, \(int\)1|jk_kernel<eritile_b200::Cls2010' -c 3 -o $O/top \
  python tools/profile_build.py --waters 80 --builds 1 --set 1000=fstrip_a_t768 --set 0000=fstrip_k2_t768 --set 2010=lane_pl512 > $O/ncu_full.log 2>&1
echo "ncu rc=$?" >> $O/ncu_full.log; tail -2 $O/ncu_full.log
