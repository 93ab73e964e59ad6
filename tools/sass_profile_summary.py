"""Per-mnemonic and per-instruction summary of an ncu source page (ncu -i X.ncu-rep --page source --csv --print-source sass > X.csv): instruction and stall-sample shares."""
import csv, collections, sys
for name in sys.argv[1:]:
    rows=list(csv.reader(open(name)))
    hdr=rows[1]; data=rows[2:]
    iA=hdr.index("Address"); iS=hdr.index("Source"); iW=hdr.index("Warp Stall Sampling (All Samples)"); iE=hdr.index("Instructions Executed")
    tot_e=sum(int(r[iE]) for r in data); tot_w=sum(int(r[iW]) for r in data)
    print(name, "instructions", tot_e, "samples", tot_w, "n", len(data))
    byop=collections.Counter(); byopw=collections.Counter()
    for r in data:
        t=r[iS].split()
        if not t: continue
        op=t[1] if t[0].startswith("@") else t[0]
        op=op.split(".")[0]
        byop[op]+=int(r[iE]); byopw[op]+=int(r[iW])
    print(" by mnemonic (inst %, stall-sample %):")
    for op,c in byop.most_common(28): print(f"   {op:10s} {100*c/tot_e:5.1f}  {100*byopw[op]/tot_w:5.1f}")
    top=sorted(data,key=lambda r:-int(r[iW]))[:30]
    print(" top stalled instructions:")
    for r in top: print(f"   {r[iA][-5:]} {int(r[iW])*100/tot_w:5.1f}% exec {int(r[iE])*100/tot_e:4.2f}%  {r[iS].strip()[:60]}")
