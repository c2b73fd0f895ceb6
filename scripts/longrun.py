"""Production-length runs on one B200 as physics evidence at scale:

* 1D-1V Landau damping 128^2 (alpha = 0.01, k = 0.5) to t = 20: damping rate
  from the |E| peaks vs the Landau root -0.153359;
* 1D-1V two-stream 1024^2 to t = 30: growth rate in [10, 25] vs the
  dispersion root 0.2931724221224933;
* 2D-2V Landau 128^4 (the bench configuration), 400 CFL steps: mass and
  total-energy drift.

Diagnostics rows come from the device (Simulation.run -> DeviceDiagnostics).
Writes <outdir>/<tag>_longrun.json and a CSV per run (tag: VPFV_LONGRUN_TAG,
default r2).

    python scripts/longrun.py [outdir]
"""
import csv
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_12155_b200 import problems as P, runner as R  # noqa: E402
from paper_2410_12155_b200.diagnostics import DiagnosticsRow, fit_growth_rate, fit_peak_rate  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "profiles"
TAG = os.environ.get("VPFV_LONGRUN_TAG", "r2")
os.makedirs(out, exist_ok=True)


def run(name, setup, t_end, cadence, max_steps=10 ** 7):
    sim = R.Simulation(setup)
    t0 = time.perf_counter()
    rows = sim.run(t_end, cadence=cadence, max_steps=max_steps)
    wall = time.perf_counter() - t0
    names = [f.species for f in setup.dists]
    with open(os.path.join(out, f"{TAG}_longrun_{name}.csv"), "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(DiagnosticsRow.header(names))
        for r in rows:
            w.writerow(r.values())
    return sim, rows, wall


summary = {}
sim, rows, wall = run("landau1d", P.make_landau_1d(P.landau_spec(alpha=0.01), 128, 128), 20.0, 5)
ts, amps = [r.t for r in rows], [r.field_amplitude for r in rows]
gamma, _ = fit_peak_rate(ts, amps, (0.0, 20.0))
summary["landau1d_128"] = {"steps": sim.step_count, "wall_s": wall, "damping_rate": gamma,
                           "reference_root": -0.153359, "rel_err": abs(gamma + 0.153359) / 0.153359}

sim, rows, wall = run("twostream", P.make_problem(P.ProblemSpec("two-stream"), 1024, 1024), 30.0, 10)
ts, amps = [r.t for r in rows], [r.field_amplitude for r in rows]
gamma, _ = fit_growth_rate(ts, amps, (10.0, 25.0))
summary["twostream_1024"] = {"steps": sim.step_count, "wall_s": wall, "growth_rate": gamma,
                             "reference_root": 0.2931724221224933,
                             "rel_err": abs(gamma - 0.2931724221224933) / 0.2931724221224933}

sim, rows, wall = run("landau2d", P.make_problem(P.landau_spec(), 128, 128), 1e9, 40, max_steps=400)
m0, m1 = rows[0].mass[0][1], rows[-1].mass[0][1]
e0, e1 = rows[0].total_energy, rows[-1].total_energy
summary["landau2d_128"] = {"steps": sim.step_count, "t_end": sim.t, "wall_s": wall,
                           "mass_rel_drift": abs(m1 - m0) / abs(m0), "energy_rel_drift": abs(e1 - e0) / abs(e0)}
with open(os.path.join(out, f"{TAG}_longrun.json"), "w") as fh:
    json.dump(summary, fh, indent=1)
print(json.dumps(summary, indent=1))
