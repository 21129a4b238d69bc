import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
for i,r in enumerate(rows):
    if "Kernel Name" in r: hdr=r; start=i+1; break
ik=hdr.index("Kernel Name"); iv=hdr.index("Metric Value"); iu=hdr.index("Metric Unit")
scale={"ns":1.0,"us":1e3,"ms":1e6,"s":1e9}
started=False
for r in rows[start:]:
    k=r[ik]
    if sys.argv[2] in k: started=True
    if started: print(f"{float(r[iv].replace(',',''))*scale.get(r[iu],1.0) if r[iv] else 0:10.1f}  {k[:70]}")
