"""8 loopback ranks, small cfg2 block moving +x: print every rank's outcome per step (debugging aid)."""
import concurrent.futures as cf
import dataclasses
import os
import sys
import traceback

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_07853_b200 import mpl  # noqa: E402
from tests.test_gpu_parity import small_cfg2  # noqa: E402

sc = small_cfg2(64)
sc = dataclasses.replace(sc, v=sc.v + np.array([5.0, 0.0, 0.0]))
R = 8
cuts = np.arange(R + 1, dtype=np.int32)
grp = mpl.Group(R)


def fn(r):
    ctx = mpl.from_scene_rank(sc, r, R, cuts, device=0, group=grp)
    log = [f"rank {r}: n0={ctx.num_particles()}"]
    try:
        for s in range(5):
            st = ctx.step(sc.dt, sc.solver)
            log.append(f"  step {s}: n={ctx.num_particles()} cells={st.get('n_cells')} newton={st.get('newton_iters')}")
    except Exception as e:  # noqa: BLE001
        log.append(f"  FAILED: {e}")
        log.append(traceback.format_exc(limit=2))
    finally:
        ctx.close()
    return "\n".join(log)


with cf.ThreadPoolExecutor(R) as ex:
    futs = [ex.submit(fn, r) for r in range(R)]
    for f in futs:
        print(f.result(timeout=600), flush=True)
grp.close()
