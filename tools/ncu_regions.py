import csv, re, collections, sys
rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 and sys.argv[1].endswith(".csv") else "gpurun_out/ncusrc/src.csv")))
hdr = rows[1]; data = rows[2:]
ix = {h:i for i,h in enumerate(hdr)}
recs = []
for r in data:
    if len(r) < len(hdr): continue
    addr = int(r[ix["Address"]], 16); src = r[ix["Source"]].strip()
    m = re.match(r'(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)', src)
    op = m.group(2) if m else "?"
    recs.append((addr, op, src, int(r[ix["Instructions Executed"]] or 0), int(r[ix["Warp Stall Sampling (All Samples)"]] or 0), float(r[ix["Avg. Threads Executed"]] or 0)))
base = recs[0][0]
T = 12582912/32
regions = [(0,0xf90,"prologue+first gather"),(0xf90,0x1680,"chunk top + patch setup"),(0x1680,0x2cb0,"ring loop"),(0x2cb0,0x2f60,"patch end stores"),(0x2f60,0x3850,"next-chunk gather"),(0x3850,0x5000,"phase C")]
tot = sum(x[3] for x in recs); ts = sum(x[4] for x in recs)
for lo,hi,name in regions:
    rs = [x for x in recs if lo <= x[0]-base < hi]
    n = sum(x[3] for x in rs); s = sum(x[4] for x in rs)
    fp = sum(x[3] for x in rs if x[1].startswith(("DFMA","DMUL","DADD")))
    cls = collections.Counter()
    for x in rs:
        cls[x[1].split(".")[0]] += x[3]
    print(f"{name:24s} warp-inst/tet {n/T:6.1f} (fp64 {fp/T:5.1f})  stall-samples {100*s/ts:5.1f}%  top: " + ", ".join(f"{k}:{v/T:.1f}" for k,v in cls.most_common(9)))
print("total per tet", tot/T)
if len(sys.argv) > 1:
    lo, hi = int(sys.argv[1],16), int(sys.argv[2],16)
    for x in recs:
        if lo <= x[0]-base < hi:
            print(hex(x[0]-base), f"{x[3]/T:5.2f}", x[4], f"{x[5]:4.1f}", x[2][:70])
