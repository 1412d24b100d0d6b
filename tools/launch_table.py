"""Summarise an ncu --metrics gpu__time_duration.sum --csv log: the kernels of the LAST frame
(after the final k_decode_apply launch) with their durations."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
iN, iV, iU = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
data = rows[1:]
start = max(i for i, r in enumerate(data) if r[iN].startswith("void queen::k_decode_apply") or "k_decode_apply" in r[iN])
tot = 0.0
for r in data[start:]:
    v = float(r[iV].replace(",", ""))
    us = v / 1000 if r[iU] == "ns" else (v if r[iU] in ("us", "usecond") else v * 1000)
    tot += us
    print(f"{r[iN][:60]:62s} {us:9.1f} us")
print(f"{'total':62s} {tot:9.1f} us")
