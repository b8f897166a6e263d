"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum launch list."""
import csv, collections, sys
for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 5]
    h = rows[0]; n = h.index("Kernel Name"); v = h.index("Metric Value")
    tot = collections.defaultdict(float); cnt = collections.Counter()
    for r in rows[1:]:
        k = r[n].split("(")[0]; t = float(r[v]) / 1e3
        tot[k] += t; cnt[k] += 1
    print(f"{f}: {len(rows) - 1} launches, total {sum(tot.values()) / 1e3:.2f} ms")
    for k, t in sorted(tot.items(), key=lambda x: -x[1])[:20]:
        print(f"  {k[:42]:42s} {cnt[k]:6d} {t:11.1f} us  avg {t / cnt[k]:9.1f}")
