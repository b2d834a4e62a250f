"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list into per-kernel counts, mean
durations and shares of the summed device time (cold-cache, serialised: shares, not absolutes)."""
import collections, csv, sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr, data = rows[0], rows[1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
acc = collections.defaultdict(list)
for r in data:
    if not r[vi]:
        continue
    v = float(r[vi].replace(",", ""))
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
    acc[r[ki].split("(")[0][:60]].append(v * scale)
tot = sum(sum(v) for v in acc.values())
print(f"{'kernel':62s} {'n':>3s} {'mean_us':>12s} {'share':>7s}")
for k, v in sorted(acc.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:62s} {len(v):3d} {sum(v) / len(v):12.1f} {sum(v) / tot:7.4f}")
