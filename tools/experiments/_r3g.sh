# Final-tree evidence (dynamic strip hand-out): smoke, headline bench, reference
# arm, launch list, ncu --set full of the tuned dominant launch, BASELINE configs.
O=gpurun_out/r02_final3; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
tail -2 $O/smoke.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
head -c 300 $O/bench.json; echo
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
head -c 300 $O/bench_reference.json; echo
ERITILE_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
   --csv --log-file $O/launches.csv python bench.py --no-cpu --no-unscreened --steps 1 --warmup 3 > $O/bench_ncu.log 2>&1
echo "launches rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:jk_strip_kernel<eritile_b200::Cls1000, \(bool\)1, \(int\)1, \(int\)1' -c 1 -o $O/top1000_tuned \
   python tools/profile_build.py --waters 80 --builds 1 --tune --profile-range > $O/ncu_full.log 2>&1
echo "ncu rc=$?"
bash tools/gpu_configs.sh r02_final3/configs
