#!/bin/bash
# quick ncu metrics (time, DRAM, L2, L1) of the tile kernel at C2 dims 128 / 64 / 32
mkdir -p gpurun_out
for d in 128 64 32; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum.per_second --clock-control none -k regex:k_tile_warp$ -s 2 -c 1 --csv --log-file gpurun_out/quick_d$d.csv python bench.py --steps 3 --warmup 3 --dim $d --no-cpu-baseline --no-e2e > /dev/null 2>&1
python3 - "$d" <<'PY'
import csv, sys
d = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/quick_d{d}.csv")))
i0 = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[i0]
im, iv, iu = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
print("dim", d, "; ".join(f"{r[im]}={r[iv]} {r[iu]}" for r in rows[i0 + 1:] if len(r) > iv))
PY
done
