# in-kernel cycle accounting of the grid kernel at several L (env TPO_GRID_PROF=1)
for L in ${LS:-1 4 7 10}; do
  TPO_GRID_PROF=1 TPO_GRID_VERBOSE=1 timeout -s KILL 60 python tools/profile_kernel.py --kind gtp_grid --L $L --reps 2 2>&1 | grep -E "tpo" | tail -3 | head -2
done
