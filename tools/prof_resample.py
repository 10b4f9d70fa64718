"""One resample (a0-a4) of a config after a warm-up resample: the ncu target for the resample's launch list.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
        python tools/prof_resample.py cfg3_ppc64
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_07853_b200 import mpl, scenes  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
sc = scenes.by_name(name, 32)
ctx = mpl.from_scene(sc, 0)
ctx.resample(sc.dt)
ctx.set_particles(sc.x, sc.v, sc.F, sc.G, sc.vol, sc.mat)
t0 = time.perf_counter()
ctx.resample(sc.dt)
print(f"{name}: resample {1e3 * (time.perf_counter() - t0):.3f} ms ({os.environ.get("MPL_P2Q", "scatter")})")
ctx.close()
