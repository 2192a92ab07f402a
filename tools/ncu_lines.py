"""Executed warp-instructions per CUDA source line (ncu source page, cuda,sass view)."""
import csv
import re
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
lines = raw.splitlines()
cur_file = None
acc = defaultdict(int)
src_text = {}
last_line = None
hdr = None
for row in csv.reader(lines):
    if not row:
        continue
    if row[0] == "File Path":
        cur_file = row[1].split("/")[-1]
        continue
    if row[0] in ("Function Name",):
        continue
    if row[0] == "Line No":
        hdr = row
        ei = hdr.index("Instructions Executed")
        continue
    if hdr is None:
        continue
    if row[0].strip():
        last_line = (cur_file, int(row[0]))
        src_text[last_line] = row[1].strip()[:90]
    # sass rows of the line: Address column non-empty
    if len(row) > ei and row[2].startswith("0x"):
        try:
            acc[last_line] += int(row[ei])
        except ValueError:
            pass
    elif len(row) > ei and row[ei].isdigit() and row[0].strip():
        acc[last_line] += int(row[ei])
tot = sum(acc.values())
print(f"total {tot:.4e}")
for k, v in sorted(acc.items(), key=lambda x: -x[1])[:top]:
    print(f"{v:13d} {v / tot:6.1%}  {k[0]}:{k[1]:4d}  {src_text.get(k, '')}")
