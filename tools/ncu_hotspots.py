import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu","-i",rep,"--page","source","--csv","-k","regex:"+kern], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
hi=[i for i,x in enumerate(r) if 'Source' in x and 'Address' in x][0]
hdr=r[hi]
i_src=hdr.index('Source'); i_s=hdr.index('Warp Stall Sampling (All Samples)'); i_n=hdr.index('Instructions Executed')
rows=[]
for x in r[hi+1:]:
    if len(x)!=len(hdr): continue
    try: rows.append((int(x[i_s] or 0), int(x[i_n] or 0), x[i_src]))
    except ValueError: pass
tot=sum(a for a,_,_ in rows)
print(kern, 'total samples',tot, 'instr', sum(n for _,n,_ in rows))
for a,n,s in sorted(rows,key=lambda t:-t[0])[:int(sys.argv[3]) if len(sys.argv)>3 else 20]: print(' ',a, n, s)
