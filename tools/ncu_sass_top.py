"""Per-SASS-instruction warp-stall samples of an ncu report (dev tool; see profiles/README.md)."""
import csv, io, subprocess, sys
path, lo, hi = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
out = subprocess.run(["ncu","-i",path,"--page","source","--csv","--print-source","sass"],capture_output=True,text=True).stdout
hdr=None; rows=[]
for ln in csv.reader(io.StringIO(out)):
    if ln and ln[0]=="Address": hdr=ln; continue
    if hdr is None or not ln: continue
    rows.append(ln)
si = hdr.index("Warp Stall Sampling (All Samples)"); src = hdr.index("Source"); ie = hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[si] or 0) for r in rows)
sel = [(float(r[si] or 0), i, r) for i, r in enumerate(rows) if lo <= i <= hi]
sel.sort(reverse=True)
for s, i, r in sel[:int(sys.argv[4]) if len(sys.argv) > 4 else 25]:
    st = sorted(((float(r[c] or 0), hdr[c][6:]) for c in stall_cols), reverse=True)[:2]
    print(f"{i:5d} {100*s/tot:5.2f}% exec={float(r[ie] or 0)/1e6:7.1f}M {' '.join(f'{n}={100*v/max(s,1):.0f}%' for v,n in st if v>0):32s} {r[src].strip()[:70]}")
