"""Join an ncu SASS source page (per-instruction counts) with nvdisasm -g line
info, and print instructions/stalls per CUDA source line.

    python scripts/sass_lines.py SASS_CSV NVDISASM_TXT KERNEL_MANGLED CELLS [MAIN_FILE]

Lines of MAIN_FILE (default stage2d2v_tma.cu) print as is; lines of every
other file (inlined helpers) print offset by 100000.
"""
import collections
import csv
import re
import sys


def main():
    sass_csv, dis, kern, cells = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
    rows = list(csv.reader(open(sass_csv)))
    h = rows[1]
    idx = {k: i for i, k in enumerate(h)}
    recs = [r for r in rows[2:] if len(r) >= len(h) and r[0].startswith("0x")]
    base = int(recs[0][idx["Address"]], 16)
    counts = {}
    for r in recs:
        off = int(r[idx["Address"]], 16) - base
        counts[off] = (int(r[idx["Instructions Executed"]] or 0), int(r[idx["Warp Stall Sampling (All Samples)"]] or 0),
                       r[idx["Source"]].strip())
    # line info from nvdisasm -g
    inside = False
    line = None
    offline = {}
    for ln in open(dis):
        if ln.startswith("\t.text.") or ln.startswith(".text."):
            inside = kern in ln
        if not inside:
            continue
        m = re.search(r'line (\d+)', ln)
        if "//##" in ln and m:
            f = re.search(r'File "([^"]+)"', ln)
            # lines of other files (tma.cuh, common.cuh helpers) are keyed apart
            line = int(m.group(1)) + (0 if not f or f.group(1).endswith(sys.argv[5] if len(sys.argv) > 5
                                                                        else "stage2d2v_tma.cu") else 100000)
            continue
        m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s', ln)
        if m and line is not None:
            offline[int(m.group(1), 16)] = line
    per = collections.defaultdict(lambda: [0, 0, collections.Counter()])
    for off, (n, st, src) in counts.items():
        l = offline.get(off, -1)
        per[l][0] += n
        per[l][1] += st
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        per[l][2][op.split(".")[0]] += n
    tot = sum(v[0] for v in per.values())
    for l in sorted(per):
        n, st, ops = per[l]
        if n == 0:
            continue
        print(f"{l:5d} {n * 32 / cells:7.2f}/cell stall={st:6d}  " +
              " ".join(f"{k}:{v * 32 / cells:.1f}" for k, v in ops.most_common(5)))
    print("total/cell", tot * 32 / cells)


if __name__ == "__main__":
    main()
