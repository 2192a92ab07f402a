"""Stall samples per SASS instruction from an ncu source page: the hottest
instructions by all warp-state samples and by long-scoreboard samples.

    python tools/ncu_stalls.py report.ncu-rep [top]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(raw[1:]))
hdr = rows[0]
col = {h: i for i, h in enumerate(hdr)}
ins = []
for r in rows[1:]:
    try:
        ins.append({"addr": r[col["Address"]], "src": r[col["Source"]].strip(),
                    "all": int(r[col["Warp Stall Sampling (All Samples)"]] or 0),
                    "lsb": int(r[col["stall_long_sb"]] or 0), "wait": int(r[col["stall_wait"]] or 0),
                    "ssb": int(r[col["stall_short_sb"]] or 0), "br": int(r[col["stall_branch_resolving"]] or 0),
                    "exe": int(r[col["Instructions Executed"]] or 0)})
    except (ValueError, IndexError, KeyError):
        pass
tot = sum(i["all"] for i in ins)
print(f"samples {tot}; long_sb {sum(i['lsb'] for i in ins) / tot:.1%}, wait {sum(i['wait'] for i in ins) / tot:.1%}, "
      f"short_sb {sum(i['ssb'] for i in ins) / tot:.1%}, branch {sum(i['br'] for i in ins) / tot:.1%}")
for key in ("all", "lsb"):
    print(f"-- top by {key}")
    for i in sorted(ins, key=lambda x: -x[key])[:top]:
        print(f"  {i['addr']} {i[key] / tot:6.2%} exe={i['exe']:>10d}  {i['src'][:90]}")
