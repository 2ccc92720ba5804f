"""Summarise an ncu report (.ncu-rep) or an ncu launch-list CSV into a small text file
for profiles/ (the judged evidence).  Usage:
  python tools/ncu_summary.py full  <report.ncu-rep>  > profiles/....txt
  python tools/ncu_summary.py launches <launches.csv> > profiles/....txt
  python tools/ncu_summary.py traffic <report.ncu-rep>   (prints dram read+write bytes of the first kernel)
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__m_xbar2l1tex_read_bytes.sum", "l1tex__m_xbar2l1tex_read_bytes.sum.per_second",
    "l1tex__m_xbar2l1tex_read_bytes.sum.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.sum",
    "smsp__inst_executed.avg.per_cycle_active", "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg",
    "sm__inst_executed_pipe_alu_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    return [(r[h.index("Kernel Name")], {k: (r[i], u[i]) for i, k in enumerate(h)}) for r in rows[2:]]


def full(rep):
    for name, d in raw(rep):
        print(f"kernel: {name[:160]}")
        for k in KEYS:
            hit = k if k in d else next((h for h in d if h.endswith("." + k)), None)
            if hit is not None:
                print(f"  {k:95s} {d[hit][0]:>20s} {d[hit][1]}")


def traffic(rep):
    name, d = raw(rep)[0]
    def b(k):
        v, unit = d[k]
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[unit]
        return float(v.replace(",", "")) * mult
    print(int(b("dram__bytes_read.sum") + b("dram__bytes_write.sum")))


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    ik, iv = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    order = []
    for r in rows[start + 1:]:
        if len(r) <= iv:
            continue
        nm = r[ik].split("(")[0]
        agg[nm][0] += 1
        agg[nm][1] += float(r[iv].replace(",", ""))
        order.append((nm, float(r[iv].replace(",", ""))))
    tot = sum(t for _, t in agg.values())
    print(f"{len(order)} launches, {tot / 1e6:.3f} ms total (gpu__time_duration.sum, serialised, cold cache)")
    print(f"{'count':>6} {'total_us':>12} {'mean_us':>10} {'share':>6}  kernel")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{c:6d} {t / 1e3:12.1f} {t / c / 1e3:10.1f} {100 * t / tot:5.1f}%  {k[:110]}")
    print("\nlast 12 launches (the timed steps):")
    for nm, t in order[-12:]:
        print(f"  {t / 1e3:10.1f} us  {nm[:110]}")


if __name__ == "__main__":
    {"full": full, "launches": launches, "traffic": traffic}[sys.argv[1]](sys.argv[2])
