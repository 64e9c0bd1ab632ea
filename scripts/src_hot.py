"""Hottest source lines of an ncu source export (--print-source cuda,sass --csv):
stall samples per line with the top stall reasons.  Usage: python scripts/src_hot.py <csv> [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
lines, fname, hdr = [], "?", None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("", "Function Name") or len(r) < len(hdr):
        continue
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ie = hdr.index("Instructions Executed")
    try:
        s = float(r[si] or 0)
    except ValueError:
        continue
    st = {hdr[i][6:]: float(r[i] or 0) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h}
    lines.append((s, fname, r[0], r[1].strip()[:80], int(float(r[ie] or 0)), st))
tot = sum(x[0] for x in lines) or 1.0
print("total samples", tot)
for s, f, ln, src, ex, st in sorted(lines, key=lambda x: -x[0])[:N]:
    top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{100 * s / tot:5.1f}% {f}:{ln:<5} ex={ex:>9} {src:80s} " + " ".join(f"{k}={100 * v / max(s, 1):.0f}" for k, v in top))
