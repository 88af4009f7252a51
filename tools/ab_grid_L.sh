# same-box A/B of grid launches at every L: base library (libtpo_b200_base.so) vs current, interleaved
for rep in 1 2; do
  echo "base $(TPO_LIB_PATH=paper_2506_13523_b200/libtpo_b200_base.so python tools/grid_time.py ${LS:-1 2 3 4 5 6 7 8 9 10} 2>&1 | grep -o '"ms": [0-9.]*' | tr '\n' ' ')"
  echo "cur  $(python tools/grid_time.py ${LS:-1 2 3 4 5 6 7 8 9 10} 2>&1 | grep -o '"ms": [0-9.]*' | tr '\n' ' ')"
done
