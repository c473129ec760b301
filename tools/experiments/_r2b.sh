O=gpurun_out/r02_b; mkdir -p $O
timeout 600 compute-sanitizer --tool memcheck python tools/repro_strip.py w8 > $O/repro_memcheck.log 2>&1; echo "rc=$?" >> $O/repro_memcheck.log
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/repro_strip.py w8 > $O/repro.log 2>&1; echo "rc=$?" >> $O/repro.log
timeout 1500 python -m pytest tests -q -m gpu --deselect "tests/test_gpu_parity.py::test_strip_kernels_vs_oracle[w8-cc-pvdz-1e-14-64-256]" --durations=30 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:jk_strip_kernel<eritile_b200::Cls1000, \(bool\)1, \(int\)1, \(int\)1' -c 1 -o $O/top1000 \
  python tools/profile_build.py --waters 80 --builds 1 --set 1000=fstrip_t768 > $O/ncu_full.log 2>&1
echo "ncu rc=$?" >> $O/ncu_full.log
tail -5 $O/repro.log; grep -c "ERROR SUMMARY" $O/repro_memcheck.log; grep "ERROR SUMMARY" $O/repro_memcheck.log | tail -2; tail -3 $O/pytest_gpu.log; tail -2 $O/ncu_full.log
