O=gpurun_out/r02_i; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:jk_strip_kernel<eritile_b200::Cls1010, \(bool\)1, \(int\)1, \(int\)1' -c 1 -o $O/s1010 \
  python tools/profile_build.py --waters 80 --builds 1 --set 1010=fstrip_a_t512 > $O/ncu_full.log 2>&1
echo "ncu rc=$?" >> $O/ncu_full.log; tail -2 $O/ncu_full.log
