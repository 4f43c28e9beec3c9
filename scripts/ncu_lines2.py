"""Per-source-line warp-stall samples of one kernel from an ncu report
(`--page source --print-source cuda,sass`): the lines holding most samples,
with their dominant stall reasons.
python scripts/ncu_lines2.py REPORT KERNEL [TOP]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", kern, "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
path, hdr, rows = None, None, []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit() and len(r) == len(hdr):
        rows.append((path, r))
idx = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for _, r in rows)
rows.sort(key=lambda x: -float(x[1][idx["Warp Stall Sampling (All Samples)"]] or 0))
print(f"total samples {tot:.0f}")
for path, r in rows[:top]:
    n = float(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    st = sorted(((float(r[idx[s]] or 0), s) for s in stalls), reverse=True)[:3]
    print(f"{100 * n / tot:5.1f}% {path}:{r[0]:>4} {r[1][:70]:70s} " + " ".join(f"{s[6:]}={v:.0f}" for v, s in st if v))
