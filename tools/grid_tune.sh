# empirical tiling sweep of the grid kernel: forced chunk width x group count per L (same box)
KIND=${KIND:-gtp_grid}
for L in ${LS:-5 6 7 8 9 10}; do
  for g in 1 2 3; do
    for nc in 48 64 80 96 112 128; do
      r=$(TPO_GRID_GROUPS=$g TPO_GRID_NC=$nc TPO_GRID_VERBOSE=1 timeout 60 python tools/grid_time.py $KIND $L 2>&1 | grep -E '"ms"|G=' | tr '\n' ' ')
      case "$r" in *tcgen05\"*) echo "L=$L g=$g nc=$nc $(echo $r | grep -o 'chunks=[0-9]* groups=[0-9]* zg=[0-9]* parts=[0-9]*') $(echo $r | grep -o '"ms": [0-9.]*')";; esac
    done
  done
  echo "L=$L default $(timeout 60 python tools/grid_time.py $KIND $L 2>&1 | grep -o '"ms": [0-9.]*')"
done
