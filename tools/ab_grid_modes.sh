# same-box comparison of grid-kernel modes (committed build vs current build x env modes)
run() { timeout 300 python tools/kind_timing.py 2>&1 | grep -E '"gtp_grid"' | grep -v '"L": 16' | sed "s/^/$1 /"; }
for rep in 1 2; do
  TPO_LIB_PATH=paper_2506_13523_b200/libtpo_b200_base.so run base
  TPO_GRID_PAIR=0 TPO_GRID_FBUFS=1 run s1
  TPO_GRID_PAIR=1 TPO_GRID_FBUFS=1 run p1
  TPO_GRID_PAIR=1 TPO_GRID_FBUFS=2 run p2
  TPO_GRID_PAIR=0 TPO_GRID_FBUFS=2 run s2
done
