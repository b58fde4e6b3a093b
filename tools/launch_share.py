"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
data = [dict(zip(h, r)) for r in rows[hi + 1:] if len(r) == len(h)]
tot = collections.defaultdict(float); cnt = collections.Counter()
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
for d in data:
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
    k = d["Kernel Name"][:70]; tot[k] += v; cnt[k] += 1
T = sum(tot.values())
print(f"| kernel | launches | total ms | avg ms | share |\n|---|---|---|---|---|")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:12]:
    print(f"| `{k}` | {cnt[k]} | {v:.3f} | {v / cnt[k]:.4f} | {100 * v / T:.1f}% |")
print(f"| all | {sum(cnt.values())} | {T:.3f} | | 100% |")
