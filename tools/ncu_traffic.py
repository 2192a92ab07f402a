"""Write profiles/traffic.json: DRAM bytes (read + write) per launch of the
dominant kernel, from one `ncu --set full` capture, keyed like bench.py."""
import csv
import json
import subprocess
import sys

rep, key, out = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "profiles/traffic.json"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
d = dict(zip(hdr, rows[2]))
u = dict(zip(hdr, units))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tot = sum(float(d[k].replace(",", "")) * scale[u[k]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
try:
    data = json.load(open(out))
except (OSError, ValueError):
    data = {}
data[key] = int(tot)
data.setdefault("_source", {})[key] = f"{rep}: {d['Kernel Name']} dram__bytes_read.sum + dram__bytes_write.sum"
json.dump(data, open(out, "w"), indent=1, sort_keys=True)
print(key, int(tot))
