"""Convergence diagnostics of one implicit step (per Newton iteration: ||g||/||g0||, PCG count,
line-search halvings, accepted step), e.g. cfg5B in fp32 and fp64.

    python tools/solve_diag.py --config cfg5B --precision 32 [--newton-max 20] [--eps-cg 1e-5] [--steps 1]
"""
import argparse
import dataclasses
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2602_07853_b200 import mpl, scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg5B")
    ap.add_argument("--precision", type=int, default=32)
    ap.add_argument("--newton-max", type=int, default=None)
    ap.add_argument("--eps-cg", type=float, default=None)
    ap.add_argument("--eps-newton", type=float, default=None)
    ap.add_argument("--ls-slack", type=float, default=None)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--psd", type=int, default=None, help="1: per-cell PSD-projected Hessian, 0: exact")
    ap.add_argument("--cg-max", type=int, default=None)
    a = ap.parse_args()
    t0 = time.time()
    sc = scenes.by_name(a.config, a.precision)
    solver = sc.solver
    kw = {k: v for k, v in (("newton_max", a.newton_max), ("eps_cg", a.eps_cg), ("eps_newton", a.eps_newton),
                            ("ls_slack", a.ls_slack), ("cg_max", a.cg_max),
                            ("psd", None if a.psd is None else bool(a.psd))) if v is not None}
    solver = dataclasses.replace(solver, **kw)
    t1 = time.time()
    ctx = mpl.from_scene(sc, 0)
    for s in range(a.steps):
        t2 = time.time()
        st = ctx.step(sc.dt, solver)
        t3 = time.time()
        g0 = st["grad_norm0"] or 1.0
        print(json.dumps({"config": a.config, "precision": a.precision, "step": s, "solver": dataclasses.asdict(solver),
                          "scene_s": round(t1 - t0, 1), "step_wall_s": round(t3 - t2, 3),
                          "converged": st["converged"], "newton_iters": st["newton_iters"],
                          "grad_rel": [g / g0 for g in st["grad_norms"]], "cg_iters": st["cg_iters"],
                          "ls_iters": st["ls_iters"], "alphas": st["alphas"], "neg_curv": st["neg_curv"],
                          "n_inverted_trials": st["n_inverted_trials"], "grad_norm0": st["grad_norm0"],
                          "ms_phase": st["ms_phase"], "n_free_nodes": st["n_free_nodes"]}), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
