#!/bin/bash
cd "$(dirname "$0")/.."
TPO_DEBUG_LASTERR=1 timeout 120 python tools/e2e_batch.py 2>&1 | grep -v "^  " | tail -5
TPO_DEBUG_LASTERR=1 timeout 120 python -c "
import torch, paper_2506_13523_b200 as tpo
for L in (3, 2, 1):
    B=1000
    hx=torch.randn(B,(L+1)**2).pin_memory(); hy=torch.randn(B,(L+1)**2).pin_memory(); ho=torch.empty(B,(2*L+1)**2).pin_memory()
    tpo.run_host_batch([('gtp_grid',hx,hy,ho,L,L,2*L)]); print('ok', L)
" 2>&1 | tail -5
