"""Per-CUDA-source-line instruction / stall totals from an ncu report (cuda,sass view)."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr = next(r for r in rows if r and r[0] == "Line No")
iE = hdr.index("Instructions Executed")
iS = hdr.index("Warp Stall Sampling (All Samples)")
lines = []
for r in rows:
    if r and r[0].isdigit():
        try:
            lines.append((int(r[0]), r[1].strip(), int(r[iE]), int(r[iS])))
        except ValueError:
            pass
totE = sum(l[2] for l in lines); totS = sum(l[3] for l in lines)
print(f"total inst {totE/1e6:.1f}M samples {totS}")
for ln, src, e, st in sorted(lines, key=lambda l: -l[3])[:top]:
    print(f"{ln:5d} {e/1e6:8.2f}M {100*e/totE:5.1f}% stall {100*st/totS:5.1f}%  {src[:80]}")
