for rep in 1 2 3; do
  echo "base $(TPO_LIB_PATH=paper_2506_13523_b200/libtpo_b200_base.so python tools/kind_timing.py 2>&1 | grep 'C": 128' | grep -o '"ms": [0-9.]*')"
  echo "cur  $(python tools/kind_timing.py 2>&1 | grep 'C": 128' | grep -o '"ms": [0-9.]*')"
done
