"""Per-SASS-instruction warp-stall samples of an ncu report (dev tool; see profiles/README.md)."""
import csv, io, subprocess, sys
def load(path):
    out = subprocess.run(["ncu","-i",path,"--page","source","--csv","--print-source","sass"],capture_output=True,text=True).stdout
    hdr=None; rows=[]
    for ln in csv.reader(io.StringIO(out)):
        if ln and ln[0]=="Address": hdr=ln; continue
        if hdr is None or not ln: continue
        rows.append(ln)
    return hdr, rows
hdr, rows = load(sys.argv[1])
si = hdr.index("Warp Stall Sampling (All Samples)")
src = hdr.index("Source")
ie = hdr.index("Instructions Executed")
tot = sum(float(r[si] or 0) for r in rows)
# regions split at BAR.SYNC / BAR.ARV
acc=0; start=0; insts=0
print("total", tot, "ninstr", len(rows))
for i,r in enumerate(rows):
    s=float(r[si] or 0); acc+=s
    op=r[src].strip()
    if op.startswith("BAR.") or "MEMBAR.ALL.GPU" in op or i==len(rows)-1:
        print(f"{start:5d}-{i:5d} {100*acc/tot:6.2f}%  ends at {op[:40]}  exec={float(rows[i][ie] or 0)/1e6:.1f}M")
        acc=0; start=i+1
