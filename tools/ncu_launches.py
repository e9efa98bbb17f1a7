import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None; d=collections.defaultdict(list)
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr and len(r)==len(hdr):
        rec=dict(zip(hdr,r))
        if rec.get('Metric Name')=='gpu__time_duration.sum':
            d[rec['Kernel Name'][:70]].append(float(rec['Metric Value']))
for k,v in d.items(): print(f"{k:70s} n={len(v):3d} median={sorted(v)[len(v)//2]/1e3:.1f} us")
