"""FP64 lane operations per cell per launch from an ncu SASS source page.

    python scripts/dp_ops.py REPORT.ncu-rep WORKLOAD CELLS [OUT_JSON]

Counts predicated-on thread instructions of DFMA / DMUL / DADD per kernel
launch in the report (ncu --page source --print-source sass, one section per
launch) and divides by the cells one launch updates; writes/updates
``dp_ops_per_cell[WORKLOAD]`` in OUT_JSON (default profiles/r2_stage_profile.json),
the file bench.py's fp64 roofline reads.
"""
import csv
import io
import json
import os
import subprocess
import sys


def main():
    rep, wl, cells = sys.argv[1], sys.argv[2], float(sys.argv[3])
    out = sys.argv[4] if len(sys.argv) > 4 else os.path.join(os.path.dirname(__file__), "..", "profiles",
                                                              "r2_stage_profile.json")
    uniq = []
    for k in range(64):  # one launch at a time: the page may repeat a launch's section
        txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                              "--launch-skip", str(k), "--launch-count", "1"],
                             capture_output=True, text=True).stdout
        cur, hdr = None, None
        for r in csv.reader(io.StringIO(txt)):
            if r and r[0] == "Kernel Name":
                if cur is not None:
                    break  # the first section is this launch
                cur = {"DFMA": 0, "DMUL": 0, "DADD": 0, "total": 0}
                continue
            if r and r[0] == "Address":
                hdr = r
                continue
            if cur is None or hdr is None or len(r) != len(hdr):
                continue
            d = dict(zip(hdr, r))
            src = d["Source"].strip().split()
            if not src:
                continue
            op = src[1] if src[0].startswith("@") and len(src) > 1 else src[0]
            n = int(d.get("Predicated-On Thread Instructions Executed") or 0)
            cur["total"] += int(d.get("Thread Instructions Executed") or 0)
            for key in ("DFMA", "DMUL", "DADD"):
                if op.split(".")[0] == key:
                    cur[key] += n
        if not cur or not cur["total"]:
            break
        uniq.append(cur)
    ops = [(p["DFMA"] + p["DMUL"] + p["DADD"]) / cells for p in uniq]
    try:
        with open(out) as f:
            prof = json.load(f)
    except (OSError, ValueError):
        prof = {}
    prof.setdefault("dp_ops_per_cell", {})[wl] = ops
    prof.setdefault("instructions_per_cell", {})[wl] = [p["total"] / cells for p in uniq]
    prof["how"] = ("DFMA + DMUL + DADD predicated-on thread instructions per launch / cells per launch, "
                   "from the ncu SASS source page of the stage-kernel capture (scripts/dp_ops.py)")
    prof.setdefault("source", {})[wl] = os.path.basename(rep)
    with open(out, "w") as f:
        json.dump(prof, f, indent=1)
    print(json.dumps({wl: ops}))


if __name__ == "__main__":
    main()
