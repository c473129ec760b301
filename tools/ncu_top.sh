#!/bin/bash
# ncu --set full of selected class kernels of one (H2O)_n Fock build.
# usage: tools/ncu_top.sh <tag> <regex> [waters]
TAG=$1; RX=$2; W=${3:-80}
O=gpurun_out/$TAG; mkdir -p $O
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:$RX" -c ${NCU_COUNT:-2} -o $O/top python tools/profile_build.py --waters $W --builds 1 ${PB_ARGS} > $O/ncu_full.log 2>&1
echo "ncu rc=$?" >> $O/ncu_full.log
tail -n 3 $O/ncu_full.log
