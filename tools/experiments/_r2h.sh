SETS="--set 1000=fstrip_a_t768 --set 0000=fstrip_k2_t768 --set 1010=fstrip_a_t512 --set 2000=fstrip_a_t512 --set 1100=fstrip_a_t512"
for L in liberitile_b200.so liberitile_probe1.so liberitile_probe2.so; do
  echo "== $L"; [ -f paper_2412_13203_b200/_lib/$L ] && ERITILE_LIBNAME=$L timeout 300 python tools/class_times.py $SETS
done
