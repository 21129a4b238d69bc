import collections,sys
agg=collections.defaultdict(lambda:[0,0.0])
for l in open(sys.argv[1]):
    p=l.split()
    if len(p)<5 or p[2]!='gap': continue
    name=" ".join(p[4:])[:60]; agg[name][0]+=1; agg[name][1]+=float(p[1])
for k,(c,t) in sorted(agg.items(),key=lambda x:-x[1][1])[:16]: print(f"{t:9.1f} {c:4d} {k}")
