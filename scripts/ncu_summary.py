"""Summarise ncu captures into profiles/ (run in the build container).

    python scripts/ncu_summary.py --launches gpurun_out/r1_launches.csv \
        --reports gpurun_out/r1_stage_s1.ncu-rep ... --out profiles/r1_summary.md --json profiles/r1_summary.json

Per stage-kernel capture it records duration, DRAM bytes (the ``traffic``
bench.py reports), pipe utilisations and stall reasons; from the launch list
(``--metrics gpu__time_duration.sum``) the per-kernel share of one step.
"""

import argparse
import collections
import csv
import io
import json
import subprocess

KEYS = {
    "duration_ms": "gpu__time_duration.sum",
    "dram_read_GB": "dram__bytes_read.sum",
    "dram_write_GB": "dram__bytes_write.sum",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smem_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
}


SCALE = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3,  # -> GB
         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,           # -> ms
         "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}


def raw(report):
    """Metric values of every profiled launch in a report (one dict each),
    bytes in GB and times in ms."""
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(io.StringIO(out))
    h = next(r)
    units = next(r)
    launches_ = []
    for vals in r:
        d = {}
        for k, u, v in zip(h, units, vals):
            if u in SCALE and v not in ("", "n/a"):
                try:
                    v = str(float(v.replace(",", "")) * SCALE[u])
                except ValueError:
                    pass
            d[k] = v
        launches_.append(d)
    return launches_


def stalls(d, n=6):
    rows = []
    for k, v in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                rows.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    return [(name, round(v, 3)) for v, name in sorted(rows, reverse=True)[:n]]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    idx = {k: i for i, k in enumerate(h)}
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[idx["Kernel Name"]].split("(")[0]
        scale = 1e-6 if r[idx["Metric Unit"]] == "ns" else (1e-3 if r[idx["Metric Unit"]] == "us" else 1.0)
        agg.setdefault(name, []).append(float(r[idx["Metric Value"]]) * scale)
    tot = sum(sum(v) for v in agg.values())
    return [dict(kernel=k, launches=len(v), total_ms=round(sum(v), 4), share=round(sum(v) / tot, 4))
            for k, v in agg.items()]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--reports", nargs="*", default=[])
    ap.add_argument("--labels", nargs="*")
    ap.add_argument("--out", required=True)
    ap.add_argument("--json", required=True)
    ap.add_argument("--title", default="ncu summary")
    ap.add_argument("--cells", type=float, default=128 ** 4)
    args = ap.parse_args()
    caps = [d for rep in args.reports for d in raw(rep)]  # every launch of every report, in order
    labels = args.labels or [f"capture {i}" for i in range(len(caps))]
    summary = {"captures": [], "launch_list": launches(args.launches) if args.launches else None}
    lines = [f"# {args.title}", ""]
    for lab, d in zip(labels, caps):
        row = {k: (float(d[v]) if v in d and d[v] not in ("", "n/a") else None) for k, v in KEYS.items()}
        row["label"] = lab
        row["kernel"] = d.get("Kernel Name", "")[:90]
        row["traffic_bytes"] = (row["dram_read_GB"] + row["dram_write_GB"]) * 1e9 if row["dram_read_GB"] is not None else None
        row["stalls"] = stalls(d)
        summary["captures"].append(row)
        lines += [f"## {lab}", f"kernel `{row['kernel']}`", "",
                  "| metric | value |", "|---|---|"]
        lines += [f"| {k} | {row[k]} |" for k in KEYS]
        lines += [f"| traffic (bytes/launch) | {row['traffic_bytes']:.4g} |",
                  f"| traffic / cell | {row['traffic_bytes'] / args.cells:.2f} B |",
                  f"| top stalls (per issue) | {', '.join(f'{n} {v}' for n, v in row['stalls'])} |", ""]
    if summary["launch_list"]:
        lines += ["## launch list (cold-cache, serialised: compare shares)", "",
                  "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        lines += [f"| `{r['kernel']}` | {r['launches']} | {r['total_ms']} | {100 * r['share']:.1f}% |"
                  for r in summary["launch_list"]]
    open(args.out, "w").write("\n".join(lines) + "\n")
    json.dump(summary, open(args.json, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
