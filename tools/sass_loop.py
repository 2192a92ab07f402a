"""Static SASS of a kernel's hot loop: the instructions between the target of the
last backward branch that encloses the VIADD.16x2 cell instructions and that branch.
usage: python tools/sass_loop.py <lib.so> <mangled-name-substring> [--list]"""
import re
import subprocess
import sys
from collections import Counter

lib, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
body = [f for f in funcs if f.split("\n")[0].strip().endswith(pat) or pat in f.split("\n")[0]]
if not body:
    sys.exit("no function matches")
f = body[0]
name = f.split("\n")[0].strip()
ins = []
for line in f.split("\n"):
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = [a for a, _ in ins]
cells = [a for a, s in ins if "VIADD.16x2" in s or "IADD.16x2" in s]
if not cells:
    sys.exit("no packed cell instructions")
lo, hi = min(cells), max(cells)
best = None
for a, s in ins:
    m = re.search(r"BRA\s+(?:!?U?P\d+,\s*)?(0x[0-9a-f]+)", s)
    if m:
        t = int(m.group(1), 16)
        if t <= lo and a >= hi:
            if best is None or (a - t) < (best[1] - best[0]):
                best = (t, a)
t, b = best
loop = [(a, s) for a, s in ins if t <= a <= b]
print(f"{name}\nloop {t:#x}..{b:#x}: {len(loop)} instructions")
c = Counter()
for a, s in loop:
    op = s.split()[0]
    if op.startswith("@"):
        op = s.split()[1]
    c[op.split(".")[0]] += 1
print(" ".join(f"{k}:{v}" for k, v in c.most_common()))
if "--list" in sys.argv:
    for a, s in loop:
        print(f"{a:6x}  {s}")
