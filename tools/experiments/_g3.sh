O=gpurun_out/r02_ncu1; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:Cls1000, \(int\)1, \(int\)1,|Cls0000, \(int\)1, \(int\)1,|jk_kernel<eritile_b200::Cls1010' -c 3 -o $O/top \
  python tools/profile_build.py --waters 80 --builds 1 --set 1000=fam_x768 --set 0000=fam_pl768 --set 1010=lane_pl512 > $O/ncu_full.log 2>&1
echo "ncu rc=$?" >> $O/ncu_full.log
tail -3 $O/ncu_full.log
