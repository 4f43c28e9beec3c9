"""Per-source-line warp instructions executed and stall samples of one
kernel launch in an ncu report.  python scripts/ncu_lines.py rep idx [n]"""
import csv
import io
import subprocess
import sys

rep, idx = sys.argv[1], int(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
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
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if hdr and r[0].isdigit() and len(r) > 6:
        try:
            ex = int(r[hdr["Instructions Executed"]] or 0)
            samp = int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        except (ValueError, KeyError):
            continue
        rows.append((ex, samp, fname, r[0], r[1].strip()[:90]))
tot = sum(x[0] for x in rows) or 1
print(f"total warp instructions {tot}")
for ex, s, f, ln, src in sorted(rows, reverse=True)[:n]:
    print(f"{100 * ex / tot:5.1f}% {ex:>10} samp={s:>5} {f}:{ln:>4} | {src}")
