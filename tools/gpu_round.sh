#!/bin/bash
# One GPU session: parity tests, bench line, ncu launch list + full capture of
# the top kernel. Outputs under gpurun_out/<tag>/.
TAG=${1:-r01}
KERN=${2:-Cls1000}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
   python bench.py --no-cpu --steps 1 --warmup 1 > $O/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KERN -c 1 -o $O/top \
   python tools/profile_build.py --waters 80 --builds 1 > $O/ncu_full.log 2>&1
ls -la $O
tail -3 $O/pytest_gpu.log; cat $O/bench.json | head -c 3000
