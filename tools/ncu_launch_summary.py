"""Summarise an ncu --csv launch list: per-kernel count, device time (us), DRAM MB, instructions."""
import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None; data=[]
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
per=collections.defaultdict(dict)
names={}
for d in data:
    v=float(d['Metric Value'].replace(',',''))
    u=d['Metric Unit']; m=d['Metric Name']
    if m=='gpu__time_duration.sum':
        v = v/1000 if u in ('nsecond','ns') else (v*1000 if u in ('msecond','ms') else v)
    if m.startswith('dram'):
        v = v/1e6 if u in ('byte','B') else (v/1e3 if u in ('Kbyte','KB') else (v if u in ('Mbyte','MB') else v*1e3))
    per[d['ID']][m]=v; names[d['ID']]=d['Kernel Name'].split('(')[0][:50]
agg=collections.defaultdict(lambda:[0,0.0,0.0,0.0])
for i,mm in per.items():
    a=agg[names[i]]; a[0]+=1; a[1]+=mm.get('gpu__time_duration.sum',0); a[2]+=mm.get('dram__bytes_read.sum',0)+mm.get('dram__bytes_write.sum',0); a[3]+=mm.get('smsp__inst_executed.sum',0)
tot=sum(v[1] for v in agg.values())
print(f"{'kernel':50s} {'n':>4s} {'us_total':>10s} {'us_avg':>9s} {'MB_avg':>9s} {'Minst_avg':>9s}")
for k,v in sorted(agg.items(), key=lambda x:-x[1][1])[:int(sys.argv[2]) if len(sys.argv)>2 else 30]:
    print(f"{k:50s} {v[0]:4d} {v[1]:10.1f} {v[1]/v[0]:9.1f} {v[2]/v[0]:9.1f} {v[3]/v[0]/1e6:9.2f}")
print('total us', tot)
