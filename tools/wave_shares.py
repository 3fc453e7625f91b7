import csv, collections, sys
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>14 and r[0]!='ID']
agg=collections.OrderedDict()
for r in rows:
    k=r[4].split('(')[0].replace('void ','')
    k=k.split('::')[-1] if 'wave_' in k else k
    a=agg.setdefault(k[:60],[0,0.0]); a[0]+=1; a[1]+=float(r[14])
tot=sum(a[1] for a in agg.values())
for k,a in sorted(agg.items(), key=lambda x:-x[1][1]):
    print(f"{k:62s} {a[0]:5d} {a[1]/1e6:9.2f} ms {100*a[1]/tot:6.2f}%")
