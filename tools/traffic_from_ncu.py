#!/usr/bin/env python
"""Write profiles/<round>/traffic.json: mean DRAM bytes (read + write) per launch of each
tcgen05 kernel kind, from an `ncu --set full` capture of one bench step
(kinds by template arguments: <0,..> fwd, <1,..> dx, <2,..> dm; a trailing `true` = the
chained pair: fwd_chain / dx_chain; roast_mix_sm100 = the fused backward: bwd_fused), and each
kind's tensor-pipe active share.  bench.py reports the bytes as roofline.traffic."""
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
itc = hdr.index("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed") \
    if "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed" in hdr else None
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
kinds = {"<0,": "fwd", "<1,": "dx", "<2,": "dm"}
acc, tpa = {}, {}
for r in rows[2:]:
    name = r[iname].replace(" ", "")
    if "roast_mix_sm100" in name:
        kind = "bwd_fused"
    else:
        kind = next((v for k, v in kinds.items() if k in name), None)
        if kind is None:
            continue
        targs = name[name.index("<") + 1:name.index(">")].split(",")
        if len(targs) >= 4 and targs[3] in ("1", "true"):
            kind += "_chain"
    b = float(r[ir]) * scale[units[ir]] + float(r[iw]) * scale[units[iw]]
    acc.setdefault(kind, []).append(b)
    if itc is not None:
        tpa.setdefault(kind, []).append(float(r[itc]))
res = {k: sum(v) / len(v) for k, v in acc.items()}
res.update({k + "_tensor_pct_active": sum(v) / len(v) for k, v in tpa.items()})
res["source"] = rep
json.dump(res, open(out, "w"), indent=1)
print(res)
