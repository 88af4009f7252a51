"""Stall breakdown of an ncu source-page CSV (--page source --csv --print-source sass),
split into regions delimited by marker instructions; prints per-region stall reasons."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
# several kernels / sections in one export: keep the first
ends = [i for i, r in enumerate(data) if r and r[0] in ("Kernel Name", "Address")]
data = data[: ends[0]] if ends else data
ia, isrc, iss = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
iex = hdr.index("Instructions Executed")
st = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
idx = [hdr.index(h) for h in st]
tot = sum(float(r[iss] or 0) for r in data)
print("total samples", tot)
# regions: runs of rows between big gaps of zero execution are not tracked; instead bucket by opcode class
# and list the top instructions with their dominant stall reason
data2 = sorted(data, key=lambda r: -float(r[iss] or 0))
for r in data2[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    reasons = sorted(((float(r[j] or 0), st[k][6:]) for k, j in enumerate(idx)), reverse=True)[:2]
    print(f"{int(r[ia], 16) & 0xFFFFF:06x} {float(r[iss]) / tot * 100:5.1f}% ex={r[iex]:>8s} {r[isrc][:70]:70s} "
          + " ".join(f"{n}:{v:.0f}" for v, n in reasons))
