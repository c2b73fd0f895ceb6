"""Quick look at one ncu --set full report: key throughputs, stalls, instruction mix per cell.

    python scripts/ncu_quick.py REPORT CELLS
"""
import collections
import csv
import io
import subprocess
import sys

rep, cells = sys.argv[1], float(sys.argv[2])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
d = dict(zip(r[0], r[2]))
for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
          "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
          "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
          "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct", "l1tex__m_xbar2l1tex_read_bytes.sum"]:
    print(f"  {k:80s} {d.get(k)}")
st = [(float(v), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]) for k, v in d.items()
      if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
print("  stalls", [(n, round(v, 2)) for v, n in sorted(st, reverse=True)[:9]])
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                      text=True).stdout
rows = list(csv.reader(io.StringIO(sass)))
h = rows[1]
idx = {k: i for i, k in enumerate(h)}
agg = collections.Counter()
tot = 0
for x in rows[2:]:
    if len(x) < len(h):
        continue
    src = x[idx["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    n = int(x[idx["Instructions Executed"]] or 0)
    agg[op.split(".")[0]] += n
    tot += n
print("  per cell:", " ".join(f"{k}:{v * 32 / cells:.1f}" for k, v in agg.most_common(22)))
print(f"  total/cell {tot * 32 / cells:.1f}")
