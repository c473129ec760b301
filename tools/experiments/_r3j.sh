# Whole-build A/B of strip vs lane variants for the mid-L classes (L2 atomic load).
O=gpurun_out/r03j; mkdir -p $O
timeout 1500 python tools/build_ab.py --waters 80 --ab 2010=strip_p_t512 --ab 2010=strip_a_t512 \
  --ab 2010=strip_p_t512,2110=strip_t512 --ab 1110=lane_pl384 --ab 2100=lane_pl512 > $O/ab.txt 2>&1
cat $O/ab.txt
