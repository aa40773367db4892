"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel count, time, share."""
import collections
import csv
import sys

path = sys.argv[1]
rows = [r for r in csv.reader(open(path)) if r]
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
ui = hdr.index("Metric Unit")
tot = collections.Counter()
cnt = collections.Counter()
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].replace("void ", "")
    v = float(r[vi].replace(",", ""))
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(r[ui], 1.0)
    tot[name] += v * scale
    cnt[name] += 1
all_ms = sum(tot.values())
print(f"| kernel | launches | total ms | share | avg ms |")
print(f"|---|---:|---:|---:|---:|")
for name, ms in tot.most_common():
    print(f"| `{name}` | {cnt[name]} | {ms:.2f} | {100 * ms / all_ms:.1f}% | {ms / cnt[name]:.4f} |")
print(f"| **all** | {sum(cnt.values())} | {all_ms:.2f} | 100% | |")
