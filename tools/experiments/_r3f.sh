# Full headline J/K parity: tuned GPU build vs one complete CPU reference build.
O=gpurun_out/r03f; mkdir -p $O
nproc > $O/nproc.txt
timeout 2400 python tools/headline_parity.py --out $O/headline_parity.json > $O/headline_parity.log 2>&1; echo "rc=$?" >> $O/headline_parity.log
tail -25 $O/headline_parity.log
