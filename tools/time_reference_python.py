"""Time the reference's own Python implementation of the hot path (SURVEY.md
8(d) "CPU baseline") in THIS container, where /root/reference exists.  The
reference cannot travel to the GPU box, so bench.py's reference arm times the
bit-exact C port instead; this script records what the real reference does on
this host's cores for the same configs, for DESIGN.md.

    PYTHONDONTWRITEBYTECODE=1 python tools/time_reference_python.py > profiles/r01_reference_python_cpu.json

Test/measurement infrastructure only: it imports the reference read-only and
never touches the product package.
"""

from __future__ import annotations

import json
import os
import sys
import time

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

import hepkit as ref  # noqa: E402


def best_of(fn, reps: int) -> float:
    best = float("inf")
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t)
    return best


def main() -> None:
    cores = os.cpu_count() or 1
    M, ms = 5.27966, (3.0969, 0.493677, 0.13957039)
    spec, mother = ref.DecaySpec(M, ms), ref.FourVector.at_rest(M)
    out = {"host_cores": cores, "how": "best-of-N wall clock, reference hepkit from /root/reference/pkg/src",
           "configs": {}}
    for workers in (1, cores):
        # C1: 1e5 events; C2 scaled to 1e7 events (a rate; 1e8 needs ~10 GB and minutes)
        for n, name, reps in ((100_000, "C1", 3), (10_000_000, "C2_rate_1e7", 1)):
            s = best_of(lambda: ref.phsp_generate(spec, mother, n, ref.RngKey(1, 1), workers=workers), reps)
            out["configs"][f"{name}_workers{workers}"] = {"events": n, "seconds": s, "events_per_s": n / s}
        # C3: chain at 1e6 (rate)
        n = 1_000_000
        sub = ref.DecaySpec(3.0969, (0.1056583755, 0.1056583755))
        blk = ref.phsp_generate(spec, mother, n, ref.RngKey(1, 1), workers=workers)
        s = best_of(lambda: ref.phsp_decay_chain(blk, 1, sub, ref.RngKey(2, 1), workers=workers), 1)
        out["configs"][f"C3_chain_step_workers{workers}"] = {"events": n, "seconds": s, "events_per_s": n / s,
                                                            "note": "phsp_decay_chain on a stored block"}

        # C5 rate: phsp_average of m12^2 over a stored 1e6 block (generation timed above)
        def m12(cols):
            e = cols["p1_e"] + cols["p2_e"]
            px = cols["p1_px"] + cols["p2_px"]
            py = cols["p1_py"] + cols["p2_py"]
            pz = cols["p1_pz"] + cols["p2_pz"]
            return (e * e - px * px - py * py - pz * pz,)

        s = best_of(lambda: ref.phsp_average(ref.identity(), blk, m12, workers=workers), 1)
        out["configs"][f"C5_average_step_workers{workers}"] = {"events": n, "seconds": s, "events_per_s": n / s}
        # C4: FCN per call at 1e7 events (toymodel scale=200, as cmd_bench)
        import toymodel  # the reference's test helper
        model = toymodel.build_model(scale=200)
        data = ref.generate_model_sample(model, ref.RngKey(7, 2), poisson=False)
        s = best_of(lambda: ref.nll(model, data, ["x0"], workers=workers), 2)
        out["configs"][f"C4_fcn_workers{workers}"] = {"events": len(data), "seconds_per_eval": s,
                                                      "evals_per_s": 1.0 / s}
        print(json.dumps(out["configs"]), file=sys.stderr)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
