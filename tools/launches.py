import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hi=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]
h=rows[hi]; data=rows[hi+1:]
ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); ii=h.index('ID')
agg=collections.defaultdict(dict)
for r in data:
    agg[(int(r[ii]), r[ki].split('(')[0])][r[mi]]=float(r[vi].replace(',',''))
n=int(sys.argv[2]) if len(sys.argv)>2 else 20
for (i,k),m in sorted(agg.items())[:n]:
    t=m.get('gpu__time_duration.sum',0)/1e3
    rd=m.get('dram__bytes_read.sum',0)/1e6; wr=m.get('dram__bytes_write.sum',0)/1e6
    print(f"{i:3d} {k:22s} {t:9.2f} us  read {rd:9.2f} MB  write {wr:7.2f} MB  {((rd+wr)/1e3)/(t/1e6) if t else 0:8.1f} GB/s")
