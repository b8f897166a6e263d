import csv, sys
for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 5]
    h = rows[0]; n = h.index("Kernel Name"); v = h.index("Metric Value")
    print(f)
    for r in rows[1:]:
        print("  %-45s %10.1f us" % (r[n][:45], float(r[v]) / 1e3))
