# round-2 ncu evidence: launch list of the c2 bench, full captures of the dominant kernels of every workload
set -x
export PYTHONUNBUFFERED=1
T=gpurun_out/r02p; mkdir -p $T
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $T/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras --no-graph --no-parity \
  > $T/bench_under_ncu.log 2>&1
cap() {  # name regex skip args...
  name=$1; rx=$2; sk=$3; shift 3
  timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:$rx -s $sk -c 1 \
    -o $T/$name python tools/profile_kernel.py "$@" > $T/ncu_$name.log 2>&1
}
cap grid_L10 gtp_grid_tc 2 --kind gtp_grid --L 10
cap grid_L3 gtp_grid_tc 2 --kind gtp_grid --L 3
cap grid_L8 gtp_grid_tc 2 --kind gtp_grid --L 8
cap mtp_L6 mtp_tc 2 --kind mtp --L 6
cap mtp_L10 mtp_kernel 2 --kind mtp --L 10 --batch 16384
cap cgtp_L3_c4 cgtp_edge 2 --kind cgtp --L 3 --channels 128 --batch 16384
cap cgtp_L6 cgtp_tc 2 --kind cgtp --L 6
cap cgtp_L16 cgtp_kernel 1 --kind cgtp --L 16 --batch 2048 --reps 2
cap fourier_L15 gtp_grid_tc 2 --kind gtp_fourier --L 15 --batch 16384
ls -la $T
