# ncu evidence for the kernels added late in round 1: K > 128 grid instantiation (L = 11),
# CGTP backward kernel (L = 6), CGTP blocks at L = 12; launch list of the bench
set -x
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/r01i
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r01i/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras --no-graph \
  > gpurun_out/r01i/bench_under_ncu.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:gtp_grid -s 2 -c 1 \
  -o gpurun_out/r01i/grid_L11 python tools/profile_kernel.py --kind gtp_grid --L 11 > gpurun_out/r01i/ncu_grid_L11.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:cgtp_bwd -s 1 -c 1 \
  -o gpurun_out/r01i/cgtp_bwd_L6 python tools/profile_cgtp_bwd.py > gpurun_out/r01i/ncu_cgtp_bwd.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:cgtp_tc -s 2 -c 1 \
  -o gpurun_out/r01i/cgtp_L12 python tools/profile_kernel.py --kind cgtp --L 12 --batch 16384 > gpurun_out/r01i/ncu_cgtp_L12.log 2>&1
ls -la gpurun_out/r01i
