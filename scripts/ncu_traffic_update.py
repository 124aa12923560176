"""Write per-launch DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of each conv layer
into profiles/ncu_traffic.json from gpurun_out/<cfg>_convs.ncu-rep (launch i = conv layer i)."""
import csv, json, subprocess, sys
from pathlib import Path

import os
out = Path(os.environ.get("TRAFFIC_OUT", "profiles/ncu_traffic.json"))
d = json.loads(out.read_text()) if out.exists() else {}
for c in sys.argv[1:]:
    rep = Path(f"gpurun_out/{c}_convs.ncu-rep")
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True, text=True).stdout
    rows = [r for r in csv.reader(txt.splitlines()) if r and r[0].isdigit()]
    hdr = next(r for r in csv.reader(txt.splitlines()) if r and r[0] == "ID")
    units = next(r for r in csv.reader(txt.splitlines()) if r and r[0] == "")
    ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for i, r in enumerate(rows):
        b = float(r[ir]) * scale[units[ir]] + float(r[iw]) * scale[units[iw]]
        d[f"{c.upper()}:conv{i}"] = int(round(b))
        print(c, i, r[4][:60], int(round(b)))
out.write_text(json.dumps(d, indent=1) + "\n")
