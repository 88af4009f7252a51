# CGTP backward A/B: bank-aware term order (TPO_CGTP_BWD_ORDER), window width (TPO_CGTP_BWD_W)
timeout -s KILL 500 python -m pytest tests/test_gpu_backward.py -q -rf --timeout 300 -p no:cacheprovider -k cgtp 2>&1 | tail -2
for O in 1 0; do echo "order=$O"; TPO_CGTP_BWD_ORDER=$O python tools/bwd_timing.py --kinds cgtp --Ls 2,3,4,6,8; done
