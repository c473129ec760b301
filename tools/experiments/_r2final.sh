# Round-2 evidence on the final tree: GPU tests, smoke, headline bench (with CPU
# baseline), reference arm, launch list, ncu --set full of the dominant launch,
# BASELINE configs.
O=gpurun_out/r02_final2; mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
tail -2 $O/smoke.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
head -c 400 $O/bench.json; echo
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
head -c 300 $O/bench_reference.json; echo
ERITILE_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
   --csv --log-file $O/launches.csv python bench.py --no-cpu --no-unscreened --steps 1 --warmup 3 > $O/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:jk_strip_kernel<eritile_b200::Cls1000, \(bool\)1, \(int\)1, \(int\)1' -c 1 -o $O/top1000 \
   python tools/profile_build.py --waters 80 --builds 1 --tune > $O/ncu_full.log 2>&1
echo "ncu rc=$?"; tail -1 $O/ncu_full.log
bash tools/gpu_configs.sh r02_final2/configs
