O=gpurun_out/r02_ncu2; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:jk_strip_kernel<eritile_b200::Cls1000, \(bool\)1, \(int\)1, \(int\)1' -c 1 -o $O/strip \
  python tools/profile_build.py --waters 80 --builds 1 --set 1000=fstrip_t512 > $O/ncu_full.log 2>&1
echo "ncu rc=$?" >> $O/ncu_full.log
tail -3 $O/ncu_full.log
