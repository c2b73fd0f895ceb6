"""Group the per-source-line output of sass_lines.py into code regions of the
2D-2V stage kernel (csrc/stage2d2v_tma.cu) and print instructions per cell and
the share of warp-stall samples per region.

    python scripts/stall_regions.py LINES_TXT [LINES_TXT ...]

LINES_TXT: `python scripts/sass_lines.py SASS_CSV NVDISASM_TXT KERNEL CELLS` output.
Line ranges follow the current source (update them when the kernel moves).
"""
import re
import sys

REGIONS = [  # (name, first line, last line) in csrc/stage2d2v_tma.cu (round-2 final source)
    ("upwind 6-point chains wpos/wneg (inlined into every stencil)", 131, 136),
    ("x scatter + window slide", 143, 228),
    ("TMA issue (producer lanes)", 229, 264),
    ("kernel setup, producer warpgroup", 265, 429),
    ("loop head, stage wait, tables", 430, 484),
    ("own rows: loads, D/G, x-coupled, vx/vy lines, diag", 485, 632),
    ("y arms: y lines, arm corners, fold", 633, 672),
    ("finalise: RK combination, stores", 673, 714),
    ("finalise: moment partials + non-finite", 715, 776),
    ("plane advance + empty-barrier arrive", 777, 786),
    ("inlined helpers (tma.cuh mbarrier waits, common.cuh)", 100000, 200000),
]


def parse(path):
    rows = {}
    for ln in open(path):
        m = re.match(r"\s*(-?\d+)\s+([\d.]+)/cell stall=\s*(\d+)", ln)
        if m:
            rows[int(m.group(1))] = (float(m.group(2)), int(m.group(3)))
    return rows


def main():
    for path in sys.argv[1:]:
        rows = parse(path)
        tot_i = sum(v[0] for v in rows.values())
        tot_s = sum(v[1] for v in rows.values())
        print(f"## {path}: {tot_i:.1f} thread instructions per cell")
        print("| region | instr/cell | stall samples |")
        print("|---|---|---|")
        seen = set()
        for name, a, b in REGIONS:
            ks = [k for k in rows if a <= k <= b]
            seen.update(ks)
            i = sum(rows[k][0] for k in ks)
            s = sum(rows[k][1] for k in ks)
            print(f"| {name} | {i:.1f} | {100 * s / tot_s:.1f} % |")
        rest = [k for k in rows if k not in seen]
        print(f"| other (setup, tma.cuh helpers, ...) | {sum(rows[k][0] for k in rest):.1f} | "
              f"{100 * sum(rows[k][1] for k in rest) / tot_s:.1f} % |")
        print()


if __name__ == "__main__":
    main()
