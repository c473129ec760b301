SETS="--set 2010=lane_pl384 --set 1110=lane_pl384 --set 2110=lane_plm1 --set 2111=lane_plm1 --set 2100=lane_pl512 --set 2011=lane_plm1 --set 1000=fstrip_a_t512 --set 1010=fstrip_p_t512"
for L in liberitile_b200.so liberitile_probe_nored.so; do
  [ -f paper_2412_13203_b200/_lib/$L ] || continue; echo "== $L"; ERITILE_LIBNAME=$L timeout 300 python tools/class_times.py $SETS
done
