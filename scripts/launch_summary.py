"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list (dev aid)."""
import collections, csv, io, sys

text = open(sys.argv[1]).read()
text = text[text.index('"ID"'):]
rows = list(csv.DictReader(io.StringIO(text)))
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    k = r["Kernel Name"].split("(")[0][:70]
    agg[k][0] += 1
    agg[k][1] += float(r["Metric Value"])
tot = sum(v[1] for v in agg.values())
print(f"{'launches':>8} {'total ms':>10} {'share':>7}  kernel")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[0]:8d} {v[1] / 1e6:10.3f} {100 * v[1] / tot:6.2f}%  {k}")
