"""tp_b200: the reference CLI's `run` / `bench` on the GPU.
CPU: the binary is built and prints its usage.  GPU: `run` reproduces the
reference's inputs (mt19937_64 + per-vector normal_distribution, x then y,
proj/tools/tp_main.cpp:107-110) and matches the fp64 oracle product; `bench`
emits the `tp bench` CSV schema (proj/src/bench.cpp:166-181)."""
import csv
import io
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
EXE = ROOT / "paper_2506_13523_b200" / "tp_b200"


def test_cli_built_and_usage():
    assert EXE.exists(), "build() makes paper_2506_13523_b200/tp_b200"
    r = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 2 and "tp_b200 run" in r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("kind,impl,L,L3", [("gtp", "grid", 3, 6), ("gtp", "fourier", 2, 4), ("cgtp", "sparse", 2, 0),
                                            ("mtp", "sparse", 2, 4)])
def test_cli_run_matches_oracle(orc, kind, impl, L, L3):
    r = subprocess.run([str(EXE), "run", "--kind", kind, "--impl", impl, "--L", str(L), "--seed", "20240901"],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    rows = list(csv.DictReader(io.StringIO(r.stdout)))
    vec = {n: np.array([float(q["value"]) for q in rows if q["vector"] == n]) for n in ("x", "y", "out")}
    rng = orc.Rng(20240901)
    x, y = rng.tower(L), rng.tower(L)
    assert np.array_equal(vec["x"], x) and np.array_equal(vec["y"], y)  # the reference's exact draws
    t = orc.tower(L)
    ref = {"gtp": orc.gtp_grid if impl == "grid" else orc.gtp_fourier}.get(kind)
    if kind == "cgtp":
        want = orc.cgtp_mimo(t, x, t, y)
    elif kind == "mtp":
        want = orc.mtp(t, x, t, y, L3)
    else:
        want = ref(t, x, t, y, L3)
    # fp32 device arithmetic on inputs rounded to fp32
    assert np.abs(vec["out"] - want).max() <= 1e-5 * np.abs(want).max() + 1e-6


@pytest.mark.gpu
def test_cli_bench_schema():
    r = subprocess.run([str(EXE), "bench", "--kinds", "gtp,mtp,cgtp", "--L", "2..3", "--batch", "4096",
                        "--warmup", "1", "--repeats", "5"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    rows = list(csv.DictReader(io.StringIO(r.stdout)))
    assert list(rows[0].keys()) == ["kind", "impl", "mode", "L", "batch", "ops", "time_med_ns", "time_min_ns",
                                    "time_max_ns", "expressivity", "ops_per_expr", "time_per_expr_ns"]
    assert len(rows) == 8  # gtp grid + fourier, mtp, cgtp at L = 2, 3
    for q in rows:
        assert int(q["time_min_ns"]) <= int(q["time_med_ns"]) <= int(q["time_max_ns"])
        ex = {"cgtp": sum(2 * min(a, b) + 1 for a in range(int(q["L"]) + 1) for b in range(int(q["L"]) + 1))}
        assert int(q["expressivity"]) == ex.get(q["kind"], 4 * int(q["L"]) + 1)
