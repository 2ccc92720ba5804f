"""Aggregate an ncu `--page source --print-source cuda,sass --csv` dump by CUDA source line."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
out = []
fname = "?"
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        i_s = hdr.index("Warp Stall Sampling (All Samples)")
        i_e = hdr.index("Instructions Executed")
        stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr is None or len(r) < len(hdr) or not r[0]:
        continue
    try:
        s = int(r[i_s]); e = int(r[i_e] or 0)
    except ValueError:
        continue
    st = sorted(((int(r[i] or 0), hdr[i][6:]) for i in stall_cols), reverse=True)[:2]
    out.append((s, e, f"{fname}:{r[0]}", r[1].strip()[:80], st))
tot = sum(o[0] for o in out)
texe = sum(o[1] for o in out)
print(f"samples {tot}  executed {texe/1e6:.1f}M")
for s, e, loc, src, st in sorted(out, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{s:7d} {100*s/tot:5.1f}% {e/1e6:8.2f}M {loc:22s} {src:80s} {st}")
