#!/bin/bash
# ncu captures of the separable row-quad kernel (L = 16, 13) and the SIMT MTP at L = 12
export PYTHONUNBUFFERED=1
cd /root/repo
T=gpurun_out/r02x; mkdir -p $T
cap() {  # name regex skip count script args...
  name=$1; rx=$2; sk=$3; c=$4; shift 4
  timeout -s KILL 500 ncu --set full --clock-control none --import-source on -k regex:$rx -s $sk -c $c \
    -o $T/$name python "$@" > $T/ncu_$name.log 2>&1
  echo "$name rc=$?"
}
cap quad_L16 grid_quad 2 1 tools/profile_kernel.py --kind gtp_grid --L 16 --batch 65536
cap quad_L13 grid_quad 2 1 tools/profile_kernel.py --kind gtp_grid --L 13 --batch 65536
cap mtp_L12 mtp 2 1 tools/profile_kernel.py --kind mtp --L 12 --batch 65536
ls -la $T
