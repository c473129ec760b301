# Round-2 re-entry check on the restored tree: GPU tests, smoke, headline bench,
# launch list, ncu --set full of the TUNED (ps|ss) strip launch (profile range =
# the tuned builds only).
O=gpurun_out/r02_reentry; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
tail -2 $O/smoke.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
head -c 400 $O/bench.json; echo
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:jk_strip_kernel<eritile_b200::Cls1000, \(bool\)1, \(int\)1, \(int\)1' -c 1 -o $O/top1000_tuned \
   python tools/profile_build.py --waters 80 --builds 1 --tune --profile-range > $O/ncu_full.log 2>&1
echo "ncu rc=$?"; tail -1 $O/ncu_full.log
