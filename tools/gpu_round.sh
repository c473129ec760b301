#!/bin/bash
# One GPU session: parity tests, bench line, ncu launch list + full capture of
# the top kernel (tuned variant). Outputs under gpurun_out/<tag>/.
#   tools/gpu_round.sh <tag> <kernel regex>
TAG=${1:-r01}
KERN=${2:-none}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
# launch list of the timed builds only (cudaProfilerStart/Stop around them)
ERITILE_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
   --csv --log-file $O/launches.csv python bench.py --no-cpu --no-unscreened --steps 1 --warmup 3 > $O/bench_ncu.log 2>&1
if [ "$KERN" != "none" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
     -k "regex:$KERN" -c 1 -o $O/top python tools/profile_build.py --waters 80 --builds 1 --tune > $O/ncu_full.log 2>&1
fi
ls -la $O
tail -3 $O/pytest_gpu.log; head -c 1500 $O/bench.json
