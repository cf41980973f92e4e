"""Artifact fixtures from the reference's own batch front end.

Runs ``aderdg.cli.run_simulation`` / ``convergence_study`` of the reference
(``/root/reference/pkg/src/aderdg/cli.py:196-302``) in the build container and
stores its ``metrics.csv``, ``solution_final.csv`` and ``run.json`` under
``tests/golden/cli/<case>/``; ``tests/test_gpu_cli.py`` compares the GPU
front end's artifacts with them.

    python tests/golden/make_cli_golden.py
"""

import json
import os
import shutil
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

CASES = {
    "wave_fused": dict(scenario="smooth-density-wave", mode="fused", steps=5),
    "spike_fused": dict(scenario="speed-spike", mode="fused", steps=8, spike_step=4),
    "wave_straightforward": dict(scenario="smooth-density-wave", mode="straightforward", steps=4),
    "wave_inject": dict(scenario="smooth-density-wave", mode="fused", steps=4, inject_rerun=True, L=2),
    "advect_fused_d3": dict(scenario="gaussian-advect", mode="fused", steps=6, d=3, p=2),
    "advect_sf_final_time": dict(scenario="gaussian-advect", mode="straightforward", final_time=0.02, p=3),
    "uniform_fused": dict(scenario="uniform", mode="fused", steps=2),
    "wave_forced_creeping": dict(scenario="smooth-density-wave", mode="fused", steps=6,
                                 forced_dt=2e-4, averaging="creeping", L=2, p=2),
    "sod_limiter": dict(scenario="sod", mode="straightforward", steps=20, limiter=True, L=2, p=3),
}
CONVERGENCE = {"conv_p2": (dict(scenario="gaussian-advect", d=2, p=2), (1, 2), 0.02)}


def main():
    from aderdg.cli import RunConfig, convergence_study, run_simulation, write_convergence_csv
    tmp = tempfile.mkdtemp()
    only = sys.argv[1:]
    for name, kw in CASES.items():
        if only and name not in only:
            continue
        out = os.path.join(tmp, name)
        cfg = RunConfig(out=out, **kw)
        run_simulation(cfg)
        dst = os.path.join(HERE, "cli", name)
        os.makedirs(dst, exist_ok=True)
        for f in ("metrics.csv", "solution_final.csv", "run.json"):
            shutil.copy(os.path.join(out, f), os.path.join(dst, f))
        with open(os.path.join(dst, "case.json"), "w") as fh:
            json.dump(kw, fh, indent=1)
        print(name, "ok")
    for name, (kw, levels, tf) in CONVERGENCE.items():
        if only and name not in only:
            continue
        rows = convergence_study(RunConfig(**kw), levels, final_time=tf)
        dst = os.path.join(HERE, "cli", name)
        os.makedirs(dst, exist_ok=True)
        write_convergence_csv(os.path.join(dst, "convergence.csv"), rows)
        with open(os.path.join(dst, "case.json"), "w") as fh:
            json.dump({"config": kw, "levels": levels, "final_time": tf}, fh, indent=1)
        print(name, rows)
    shutil.rmtree(tmp)


if __name__ == "__main__":
    main()
