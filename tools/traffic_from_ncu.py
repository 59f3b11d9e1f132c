#!/usr/bin/env python
"""Write profiles/<round>/traffic.json: mean DRAM bytes (read + write) per launch of each
tcgen05 kernel kind, from an `ncu --set full` capture of one bench step
(launch order fwd L1, fwd L2, dx L2, dm L2, dx L1, dm L1).  bench.py reports it as
roofline.traffic."""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
iname = hdr.index("Kernel Name")
ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
kinds = {"<0,": "fwd", "<1,": "dx", "<2,": "dm"}
acc = {}
for r in rows[2:]:
    kind = next((v for k, v in kinds.items() if k in r[iname].replace(" ", "")), None)
    if kind is None:
        continue
    b = float(r[ir]) * scale[units[ir]] + float(r[iw]) * scale[units[iw]]
    acc.setdefault(kind, []).append(b)
res = {k: sum(v) / len(v) for k, v in acc.items()}
res["source"] = rep
json.dump(res, open(out, "w"), indent=1)
print(res)
