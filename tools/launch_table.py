"""Markdown table of an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import csv, collections, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0] != 'ID']
agg = collections.OrderedDict()
for r in rows:
    k = r[4].split('(')[0].replace('void ', '')
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += float(r[14].replace(',', ''))
tot = sum(a[1] for a in agg.values())
print("| kernel | launches | total ms | share |\n|---|---:|---:|---:|")
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| `{k}` | {a[0]} | {a[1] / 1e6:.1f} | {100 * a[1] / tot:.2f}% |")
