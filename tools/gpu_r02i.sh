# (1) A/B round-1 vs current grid kernel on the c2 sweep (same box), (2) precision at L = 15, 16 for the
# tcgen05 CGTP blocks and the grid / Fourier degree groups, (3) timing of those paths at the c5 shard
export PYTHONUNBUFFERED=1
D=gpurun_out/r02i; mkdir -p $D
for lib in r01 cur r01 cur; do
  if [ $lib = r01 ]; then export TPO_LIB_PATH=$PWD/tools/ab/libtpo_r01.so; else unset TPO_LIB_PATH; fi
  timeout -s KILL 300 python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline --no-parity > $D/bench_$lib.log 2>&1
  python - $D/bench_$lib.log $lib <<'PY'
import json, sys
l = [x for x in open(sys.argv[1]) if x.startswith('{')]
if not l: print(sys.argv[2], open(sys.argv[1]).read()[-1500:]); sys.exit()
d = json.loads(l[-1])
print(sys.argv[2], round(d['value']/1e6,1), d['ms_per_step'], [round(v['ms'],4) for v in d['per_kind_L'].values()], d['roofline']['frac'])
PY
done
unset TPO_LIB_PATH
cat > /tmp/hiL.py <<'PY'
import sys, json, time, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle'); sys.path.insert(0, 'tests')
import oracle as orc, paper_2506_13523_b200 as tpo
from test_gpu_parity_scale import adversarial_rows, _normwise_rows
res = {}
for kind in ("cgtp", "gtp_grid", "gtp_fourier"):
    for L in (15, 16):
        rng = np.random.default_rng(31337 + 17 * L)
        x, y, names = adversarial_rows(L, rng, per=3)
        L3 = 0 if kind == "cgtp" else 2 * L
        out = tpo.run(kind, torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), L, L, L3).cpu().numpy()
        ref = orc.batch_mimo(kind, L, x.astype(np.float64)[:, None], y.astype(np.float64)[:, None])[:, 0]
        err = _normwise_rows(out, ref)
        path = tpo.context().last_grid_path if kind != "cgtp" else "-"
        # timing at the c5 shard (2^19 products)
        B = 1 << 19 if kind != "cgtp" else 1 << 15
        xb = torch.randn((B, (L + 1) ** 2), device="cuda"); yb = torch.randn((B, (L + 1) ** 2), device="cuda")
        tpo.run(kind, xb, yb, L, L, L3); torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); tpo.run(kind, xb, yb, L, L, L3); b.record(); b.synchronize()
        ms = a.elapsed_time(b) * ((1 << 19) / B)
        res[f"{kind}_L{L}"] = {"worst": float(err.max()), "path": path, "ms_2^19": round(ms, 2)}
        print(kind, L, res[f"{kind}_L{L}"], flush=True)
PY
for cfg in base tc; do
  if [ $cfg = tc ]; then export TPO_CGTP_TC_MAXL=16 TPO_GRID_SPLIT_MAXL=16; fi
  echo "== $cfg"; timeout -s KILL 900 python /tmp/hiL.py 2>&1 | tail -8
done
