import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
for i,r in enumerate(rows):
    if "Kernel Name" in r: hdr=r; start=i+1; break
ik=hdr.index("Kernel Name"); iv=hdr.index("Metric Value")
started=False
for r in rows[start:]:
    k=r[ik]
    if sys.argv[2] in k: started=True
    if started: print(f"{float(r[iv].replace(',','')) if r[iv] else 0:10.1f}  {k[:70]}")
