import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if hdr is None:
        if "Kernel Name" in r: hdr = {h: i for i, h in enumerate(r)}
        continue
    if len(r) < len(hdr) or r[hdr["Metric Name"]] != "gpu__time_duration.sum": continue
    k = r[hdr["Kernel Name"]].split("(")[0][:60]
    v = float(r[hdr["Metric Value"]].replace(",", ""))
    unit = r[hdr["Metric Unit"]]
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}.get(unit, 1.0)
    agg[k][0] += 1; agg[k][1] += v * scale
tot = sum(t for n, t in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:14]: print(f"{t/1000:9.2f} ms {100*t/tot:5.1f}% {n:4d}  {k}")
