"""Per-instruction execution counts from an ncu source page (SASS): opcode histogram
weighted by executed warp-instructions, and the hottest basic regions."""
import csv
import re
import subprocess
import sys
from collections import Counter

ALU = {"VIADDMNMX", "VIMNMX", "VIMNMX3", "SEL", "LOP3", "LEA", "SHF", "IADD3", "ISETP", "PRMT", "FLO",
       "BREV", "POPC", "PLOP3", "VIADD", "IABS", "FMNMX"}
FMA = {"IMAD", "IADD", "IMUL", "FFMA", "FMUL", "FADD"}


def main(path, top=40):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = raw.splitlines()
    rows = list(csv.reader(lines[1:]))
    hdr = rows[0]
    ai, si, ei = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
    ins = []
    for r in rows[1:]:
        try:
            ins.append((int(r[ai], 16), r[si].strip(), int(r[ei])))
        except (ValueError, IndexError):
            pass
    tot = sum(e for _, _, e in ins)
    op_c = Counter()
    pipe = Counter()
    for a, s, e in ins:
        op = re.sub(r"^@!?U?P\w+\s+", "", s).split()[0] if s else "?"
        base = op.split(".")[0]
        op_c[op] += e
        pipe["ALU" if base in ALU else "FMA" if base in FMA else "other"] += e
    print(f"total executed warp-instructions {tot:.3e}")
    print("pipe split (by opcode class):", {k: f"{v / tot:.1%}" for k, v in pipe.items()})
    for op, e in op_c.most_common(top):
        print(f"  {op:28s} {e:14d} {e / tot:6.1%}")
    return ins


if __name__ == "__main__":
    main(sys.argv[1])
