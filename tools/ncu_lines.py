"""Top source lines by warp-stall samples from an ncu report (cuda,sass view).

    ncu -i rep --page source --csv --print-source cuda,sass > x.csv
    python tools/ncu_lines.py x.csv [N]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None
out = []
fname = ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0].isdigit():
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        smp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    reasons = {k: int(v) for k, v in d.items() if k.startswith("stall_") or "Stall" in k and k not in (
        "Warp Stall Sampling (All Samples)", "Warp Stall Sampling (Not-issued Samples)") if v.isdigit() and int(v) > 0}
    out.append((smp, fname, r[0], r[1].strip()[:90], reasons))
tot = sum(o[0] for o in out)
out.sort(reverse=True)
print(f"total samples {tot}")
for smp, f, ln, src, rs in out[:n]:
    top = sorted(rs.items(), key=lambda kv: -kv[1])[:3]
    print(f"{100.0 * smp / tot:5.1f}% {f}:{ln:>5} {src:90s} {top}")
