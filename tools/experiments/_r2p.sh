O=gpurun_out/r02_p; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_c5.py -q -x --durations=5 > $O/pytest_c5.log 2>&1; echo "rc=$?" >> $O/pytest_c5.log
tail -4 $O/pytest_c5.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:coopw_kernel<eritile_b200::CoopCls2221|coop_kernel<eritile_b200::CoopCls3221' -c 2 -o $O/coop \
  python tools/profile_build.py --geom ala2 --basis cc-pvtz.txt --builds 1 --set 2221=coopw --set 3221=coop > $O/ncu_full.log 2>&1
echo "ncu rc=$?" >> $O/ncu_full.log; tail -2 $O/ncu_full.log
