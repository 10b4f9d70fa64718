"""Explicit-path throughput on one GPU.

    python tools/explicit_bench.py [--config jelly] [--steps 50] [--warmup 5]

Runs mpl_explicit_step (resample -> f_i = -sum V tau grad w, v += dt (g + f/m) -> G2P) back to back on
the configured scene and prints one JSON line: ms per step (CUDA events inside the library, summed over
the three phases), particle-steps per second, and the phase split.  The algorithmic particle traffic
per step (fp32: P2Q reads x, v, F, G, vol, mat = 104 B; G2P reads x, F and writes x, v, F, G = 144 B)
gives the particle-bandwidth roofline figure."""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_07853_b200 import mpl, scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="jelly")
    ap.add_argument("--precision", type=int, default=32)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    a = ap.parse_args()
    sc = scenes.by_name(a.config, a.precision)
    ctx = mpl.from_scene(sc, 0)
    for _ in range(a.warmup):
        ctx.explicit_step(sc.dt)
    ph = np.zeros(8)
    launches = 0
    for _ in range(a.steps):
        st = ctx.explicit_step(sc.dt)
        ph += np.asarray(st["ms_phase"])
        launches += st["n_launches"]
    x, v, F, G = ctx.get_particles()
    ctx.close()
    assert np.all(np.isfinite(x)) and np.all(np.isfinite(F))
    ms = ph[7] / a.steps
    s = 4 if a.precision == 32 else 8
    alg = sc.n_particles * (26 * s + 36 * s)  # 104 + 144 B in fp32
    print(json.dumps({
        "path": "explicit", "config": a.config, "precision": a.precision, "particles": sc.n_particles,
        "steps": a.steps, "ms_per_step": round(ms, 4),
        "particle_steps_per_s": round(sc.n_particles / (ms * 1e-3), 1),
        "phase_ms": {"resample": round(ph[0] / a.steps, 4), "explicit_update": round(ph[2] / a.steps, 4),
                     "g2p": round(ph[6] / a.steps, 4)},
        "launches_per_step": launches / a.steps,
        "particle_bytes_per_step": alg,
        "particle_GBps": round(alg / (ms * 1e-3) / 1e9, 1),
    }), flush=True)


if __name__ == "__main__":
    main()
