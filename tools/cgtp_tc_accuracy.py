# accuracy of the CGTP block path at L = 12..15 on rows of mixed magnitude (TPO_CGTP_TC_MAXL=16)
import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import paper_2506_13523_b200 as tpo, oracle as orc
for L, B in [(12, 40), (13, 24), (14, 16), (15, 8)]:
    for trial in range(3):
        rng = np.random.default_rng(360 + L + 100 * trial)
        x = rng.standard_normal((B, (L + 1) ** 2)).astype(np.float32); y = rng.standard_normal((B, (L + 1) ** 2)).astype(np.float32)
        x[0] *= 1e-3; y[1] *= 1e3
        out = tpo.run('cgtp', torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), L, L, 0).cpu().numpy().astype(np.float64)
        ref = orc.batch_mimo('cgtp', L, x.astype(np.float64)[:, None], y.astype(np.float64)[:, None])[:, 0]
        err = (np.abs(out - ref).max(1) / np.abs(ref).max(1)).max()
        print(L, trial, err, flush=True)
