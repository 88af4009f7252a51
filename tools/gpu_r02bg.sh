#!/bin/bash
cd /root/repo
for E in "" "TPO_GRID_PAIR=1" "TPO_GRID_GROUPS=1" "TPO_GRID_GROUPS=3" "TPO_GRID_NC=96" "TPO_GRID_NC=64" "TPO_GRID_ZG_MAX=256" "TPO_GRID_STAGES=3" "TPO_GRID_INPLACE=1" ""; do
  env $E timeout 120 python tools/grid_plan_sweep.py 8,9,10 2>&1 | tail -1
done
