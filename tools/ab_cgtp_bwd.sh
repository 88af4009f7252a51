# CGTP backward A/B: window width (TPO_CGTP_BWD_W), term split (TPO_CGTP_BWD_SPLIT)
for W in 0 256; do
  if [ $W = 0 ]; then unset TPO_CGTP_BWD_W; else export TPO_CGTP_BWD_W=$W; fi
  echo "W=$W"; python tools/bwd_timing.py --kinds cgtp --Ls 1,2,3,4,6,8
done
