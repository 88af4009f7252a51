# ncu evidence for the round: launch list of the bench command + full captures
set -x
export PYTHONUNBUFFERED=1
TAG=${TAG:-r01}
mkdir -p gpurun_out/$TAG
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/$TAG/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras --no-graph \
  > gpurun_out/$TAG/bench_under_ncu.log 2>&1
for L in ${GRID_LS:-10 8 6 1}; do
  timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:gtp_grid -s 2 -c 1 \
    -o gpurun_out/$TAG/grid_L$L python tools/profile_kernel.py --kind gtp_grid --L $L > gpurun_out/$TAG/ncu_grid_L$L.log 2>&1
done
if [ -n "$OTHERS" ]; then
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:cgtp -s 2 -c 1 \
  -o gpurun_out/$TAG/cgtp_L3_C128 python tools/profile_kernel.py --kind cgtp --L 3 --batch 16384 --channels 128 > gpurun_out/$TAG/ncu_cgtp.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:gtp_grid -s 2 -c 1 \
  -o gpurun_out/$TAG/fourier_L6 python tools/profile_kernel.py --kind gtp_fourier --L 6 > gpurun_out/$TAG/ncu_fourier.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:mtp -s 2 -c 1 \
  -o gpurun_out/$TAG/mtp_L6 python tools/profile_kernel.py --kind mtp --L 6 > gpurun_out/$TAG/ncu_mtp.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:cgtp_tc -s 2 -c 1 \
  -o gpurun_out/$TAG/cgtp_L6 python tools/profile_kernel.py --kind cgtp --L 6 > gpurun_out/$TAG/ncu_cgtp_L6.log 2>&1
fi
ls -la gpurun_out/$TAG
