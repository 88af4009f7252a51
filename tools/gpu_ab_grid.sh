# grid kernel A/B on the c2 sweep (round-1 library vs current) + PROF at L = 10 + grid/Fourier parity
export PYTHONUNBUFFERED=1
for lib in r01 cur r01 cur; do
  if [ $lib = r01 ]; then export TPO_LIB_PATH=$PWD/tools/ab/libtpo_r01.so; else unset TPO_LIB_PATH; fi
  timeout -s KILL 300 python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline --no-parity > /tmp/b_$lib.log 2>&1
  python -c "
import json,sys; d=json.loads([x for x in open('/tmp/b_$lib.log') if x.startswith('{')][-1]); print('$lib', round(d['value']/1e6,1), [round(v['ms'],4) for v in d['per_kind_L'].values()])"
done
unset TPO_LIB_PATH
TPO_GRID_PROF=1 python -c "
import torch, sys
sys.path.insert(0, '.')
import paper_2506_13523_b200 as tpo
L = 10
x = torch.randn(65536, (L+1)**2, device='cuda'); y = torch.randn(65536, (L+1)**2, device='cuda')
for _ in range(3): tpo.gtp_grid(x, y, L, L, 2*L)
torch.cuda.synchronize()
" 2>&1 | grep tpo-prof | tail -1
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -k "${TESTK:-grid or fourier or weighted or backward}" -p no:cacheprovider 2>&1 | tail -2
