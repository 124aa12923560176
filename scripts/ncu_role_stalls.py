"""Stall-reason totals per kernel role (source line ranges) from an ncu report (cuda,sass view)."""
import csv, subprocess, sys
rep = sys.argv[1]
ranges = [tuple(x.split(":")) for x in sys.argv[2:]]  # name:lo-hi
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr = next(r for r in rows if r and r[0] == "Line No")
names = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
idx = [hdr.index(h) for h in names]
iE = hdr.index("Instructions Executed")
tot = {n: [0] * len(names) for n, _ in ranges}
inst = {n: 0 for n, _ in ranges}
for r in rows:
    if not r or not r[0].isdigit():
        continue
    ln = int(r[0])
    for n, span in ranges:
        lo, hi = map(int, span.split("-"))
        if lo <= ln <= hi:
            for j, i in enumerate(idx):
                try:
                    tot[n][j] += int(r[i])
                except ValueError:
                    pass
            try:
                inst[n] += int(r[iE])
            except ValueError:
                pass
for n, _ in ranges:
    s = sum(tot[n])
    top = sorted(zip(names, tot[n]), key=lambda x: -x[1])[:6]
    print(f"{n:10s} inst {inst[n]/1e6:7.1f}M samples {s:6d}  " + "  ".join(f"{k[6:]}={100*v/max(s,1):.0f}%" for k, v in top))
