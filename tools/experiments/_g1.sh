O=gpurun_out/r02_start; mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --no-unscreened > $O/bench.json 2> $O/bench.err
tail -3 $O/pytest_gpu.log; head -c 600 $O/bench.json
