"""Summarise an ncu source-page CSV (sass): top stalls and per-landmark execution counts."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
i_s = hdr.index("Warp Stall Sampling (All Samples)"); i_src = hdr.index("Source"); i_exec = hdr.index("Instructions Executed")
stall_cols = [i for i,h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[i_s]) for r in data); texec = sum(int(r[i_exec] or 0) for r in data)
print("total samples", tot, "total executed", texec)
for r in sorted(data, key=lambda r: -int(r[i_s]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    st = sorted(((int(r[i]), hdr[i][6:]) for i in stall_cols), reverse=True)[:2]
    print(f"{r[0][-5:]} {int(r[i_s]):7d} {r[i_exec]:>10} {r[i_src][:70]:70s} {st}")
