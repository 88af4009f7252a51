# same-box A/B of the CGTP block kernel (L >= 5): base library vs current
for rep in 1 2; do
  for lib in base cur; do
    if [ $lib = base ]; then P=paper_2506_13523_b200/libtpo_b200_base.so; else P=paper_2506_13523_b200/libtpo_b200.so; fi
    echo "$lib $(TPO_LIB_PATH=$P python tools/kind_timing.py 2>&1 | grep '"cgtp"' | grep -E '"L": (4|6|8|10),' | grep -o '"ms": [0-9.]*' | tr '\n' ' ')"
  done
done
