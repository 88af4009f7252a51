# ncu --set full captures of the grid kernel at given L values (TAG, LS env)
TAG=${TAG:-v2}; mkdir -p gpurun_out/$TAG
for L in ${LS:-1 10}; do
  TPO_GRID_VERBOSE=1 timeout -s KILL 240 ncu --set full --clock-control none --import-source on -k regex:gtp_grid -s 2 -c 1 \
    -o gpurun_out/$TAG/grid_L$L python tools/profile_kernel.py --kind gtp_grid --L $L > gpurun_out/$TAG/ncu_grid_L$L.log 2>&1
done
