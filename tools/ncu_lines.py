"""Summarise an ncu source page (CUDA lines) by warp-stall samples: python tools/ncu_lines.py rep [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None; data = []
for r in rows:
    if len(r) > 3 and r[0] == "Line No":
        hdr = r; continue
    if hdr and len(r) == len(hdr) and r[0]:
        data.append(r)
ix = {h: i for i, h in enumerate(hdr)}
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data.sort(key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
print("total samples", tot)
for r in data[:N]:
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    top = sorted(((int(r[ix[h]] or 0), h[6:]) for h in stalls), reverse=True)[:3]
    print(f"{100*s/tot:5.1f}% L{r[0]:>4} {r[1].strip()[:90]:90s} " + " ".join(f"{h}={v}" for v, h in top))
