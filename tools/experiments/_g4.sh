O=gpurun_out/r02_par1; mkdir -p $O
nproc > $O/nproc.txt; lscpu | grep "Model name" >> $O/nproc.txt
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_multirank.py tests/test_gpu_parity.py -q -x --durations=15 > $O/pytest_new.log 2>&1; echo "pytest rc=$?" >> $O/pytest_new.log
tail -25 $O/pytest_new.log
