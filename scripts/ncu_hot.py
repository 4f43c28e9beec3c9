"""Top source lines / SASS of one kernel launch in an ncu report by warp-stall
samples.  python scripts/ncu_hot.py report.ncu-rep <launch-index> [n]"""
import csv
import io
import subprocess
import sys

rep, idx = sys.argv[1], int(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(idx), "--launch-count", "1",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit() and len(r) > 6:
        try:
            samp = int(r[4] or 0)
        except ValueError:
            continue
        rows.append((samp, fname, r[0], r[1].strip()[:90], r[3].strip()[:60], r[7]))
tot = sum(x[0] for x in rows) or 1
print(f"total samples {tot}")
for s, f, ln, src, sass, ex in sorted(rows, reverse=True)[:n]:
    print(f"{100*s/tot:5.1f}% {f}:{ln:>4} exec={ex:>9} | {src} | {sass}")
