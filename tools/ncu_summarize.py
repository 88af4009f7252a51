"""Summarise ncu captures (gpurun_out/<tag>/*.ncu-rep, launches.csv) into profiles/."""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

tag, out_dir = sys.argv[1], Path(sys.argv[2])
src = Path("gpurun_out") / tag
WANT = {
    "gpu__time_duration.sum": "time",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_%",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_%",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_%",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_%",
    "launch__registers_per_thread": "regs",
    "launch__shared_mem_per_block_dynamic": "dyn_smem",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_%",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3,
        "ns": 1e-3, "us": 1, "ms": 1e3, "Kbyte/block": 1e3, "byte/block": 1}
rows, traffic = [], {}
for rep in sorted(src.glob("*.ncu-rep")):
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    if len(r) < 3:
        continue
    hdr, units, vals = r[0], r[1], r[2]
    d = {"capture": rep.stem, "kernel": vals[hdr.index("Kernel Name")][:60] if "Kernel Name" in hdr else ""}
    for i, n in enumerate(hdr):
        if n in WANT:
            v = vals[i].replace(",", "")
            try:
                x = float(v) * UNIT.get(units[i], 1)
            except ValueError:
                continue
            d[WANT[n]] = x
    rows.append(d)
    if "dram_read" in d:
        traffic[rep.stem] = d["dram_read"] + d.get("dram_write", 0)
lines = ["# ncu --set full captures (%s), one launch each, cold L2 (ncu), clocks unlocked" % tag, "",
         "| capture | kernel | time us | DRAM read MB | DRAM write MB | DRAM % | tensor % | issue % | warps % | regs | dyn smem KB | grid x block | smem conflicts |",
         "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
for d in rows:
    f = lambda k, s=1, p=1: ("%.*f" % (p, d[k] / s)) if k in d else "-"
    lines.append(f"| {d['capture']} | `{d['kernel'][:40]}` | {f('time')} | {f('dram_read', 1e6)} | {f('dram_write', 1e6)} | "
                 f"{f('dram_%')} | {f('tensor_%')} | {f('issue_%')} | {f('warps_active_%')} | {f('regs', 1, 0)} | "
                 f"{f('dyn_smem', 1024, 0)} | {f('grid', 1, 0)} x {f('block', 1, 0)} | {f('smem_bank_conflicts', 1, 0)} |")
# launch list: share of device time per kernel name
ll = src / "launches.csv"
if ll.exists():
    txt = ll.read_text()
    start = txt.find('"ID"')
    rr = list(csv.DictReader(io.StringIO(txt[start:])))
    tot, per = 0.0, {}
    for x in rr:
        if x.get("Metric Name") != "gpu__time_duration.sum" or not x.get("Metric Value", "").replace(",", "").strip():
            continue
        v = float(x["Metric Value"].replace(",", "")) * UNIT.get(x.get("Metric Unit", "ns"), 1e-3)
        k = x["Kernel Name"].split("(")[0][-50:]
        per[k] = per.get(k, 0.0) + v
        tot += v
    lines += ["", "## launch list (`ncu --metrics gpu__time_duration.sum` over `bench.py --steps 3 --warmup 3`)", "",
              "| kernel | total us | share |", "|---|---|---|"]
    for k, v in sorted(per.items(), key=lambda kv: -kv[1]):
        lines.append(f"| `{k}` | {v:.1f} | {v / tot:.3f} |")
    # a timed step = the 10 grid launches between two L2-flush fills
    steps, cur = [], []
    for x in rr:
        if x.get("Metric Name") != "gpu__time_duration.sum" or not x.get("Metric Value", "").strip():
            continue
        v = float(x["Metric Value"].replace(",", "")) * UNIT.get(x.get("Metric Unit", "ns"), 1e-3)
        if "FillFunctor<float>" in x.get("Kernel Name", ""):
            if len(cur) == 10:
                steps.append(cur)
            cur = []
        elif "gtp_grid_tc_kernel" in x.get("Kernel Name", ""):
            cur.append(v)
    if steps:
        last = steps[-1]
        lines += ["", "one timed step's 10 grid launches (L = 1..10, us, ncu-serialised, cold L2): "
                  + ", ".join("%.1f" % v for v in last),
                  "share of the L=10 launch in the step: %.3f (bench, CUDA graph: see bench_v*.json share_of_step)"
                  % (last[-1] / sum(last))]
out_dir.mkdir(parents=True, exist_ok=True)
(out_dir / "ncu_summary.md").write_text("\n".join(lines) + "\n")
print("\n".join(lines))
json.dump({("gtp_grid_L" + k.split("_L")[1] if k.startswith("grid_L") else k): v for k, v in traffic.items()},
          open(out_dir.parent / "ncu_traffic.json", "w"), indent=1)
