set -x
export PYTHONUNBUFFERED=1
python tools/gpu_debug.py grid 2>&1 | tee gpurun_out/debug_grid.log
python tools/gpu_debug.py other 2>&1 | tee gpurun_out/debug_other.log
python tools/gpu_debug.py simt 2>&1 | tee gpurun_out/debug_simt.log
