"""Stall reasons summed over SASS instructions executed between LO and HI times
(ncu source page): python tools/ncu_stall_agg.py report.ncu-rep LO [HI]"""
import csv, subprocess, sys
rep=sys.argv[1]; lo=int(sys.argv[2]); hi=int(sys.argv[3]) if len(sys.argv)>3 else 10**12
raw=subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","sass"],capture_output=True,text=True).stdout.splitlines()
rows=list(csv.reader(raw[1:])); hdr=rows[0]; c={h:i for i,h in enumerate(hdr)}
reasons=[h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg={r:0 for r in reasons}; n=0; tot=0; exe=0
for r in rows[1:]:
    try: e=int(r[c["Instructions Executed"]] or 0)
    except: continue
    if "STRONG.SYS" in r[c["Source"]] or "NANOSLEEP" in r[c["Source"]]: continue
    if lo<=e<=hi:
        n+=1; exe+=e
        for k in reasons: agg[k]+=int(r[c[k]] or 0)
tot=sum(agg.values())
print("instructions",n,"executed",exe,"samples",tot)
for k,v in sorted(agg.items(),key=lambda x:-x[1])[:12]: print(f"  {k:28s} {v:8d} {v/tot:6.1%}")
