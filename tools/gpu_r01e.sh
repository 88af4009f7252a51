export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/r01e
timeout -s KILL 400 python bench.py --steps 5 --warmup 3 > gpurun_out/r01e/bench.log 2>&1
timeout -s KILL 300 python tools/bwd_timing.py > gpurun_out/r01e/bwd_timing.jsonl 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:cgtp_tc -s 2 -c 1 \
  -o gpurun_out/r01e/cgtp_L6 python tools/profile_kernel.py --kind cgtp --L 6 > gpurun_out/r01e/ncu_cgtp_L6.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:mtp -s 2 -c 1 \
  -o gpurun_out/r01e/mtp_L6 python tools/profile_kernel.py --kind mtp --L 6 > gpurun_out/r01e/ncu_mtp.log 2>&1
tail -c 600 gpurun_out/r01e/bench.log; cat gpurun_out/r01e/bwd_timing.jsonl; ls gpurun_out/r01e
