"""Input recipe checks: counts of the synthetic configs match SURVEY.md §8(d)."""
import numpy as np

from paper_2602_07853_b200 import scenes


def test_cfg1_counts_and_determinism():
    a, b = scenes.cfg1(), scenes.cfg1()
    assert a.n_particles == 4096
    assert np.array_equal(a.x, b.x) and np.array_equal(a.v, b.v)
    assert a.x.min() >= 4 / 16 and a.x.max() < 12 / 16
    c = scenes.cfg1(prestrain=True)
    assert np.all(np.linalg.det(c.F.reshape(-1, 3, 3)) > 0)
    assert not np.allclose(c.F, a.F)


def test_cfg2_counts():
    s = scenes.cfg2()
    assert s.n_particles == 884736 and s.x.dtype == np.float32
    assert s.dt == 2e-3


def test_cfg4_cfg5_cell_counts():
    n = 256
    dx = 1.0 / n
    s0 = scenes.cells_sphere(n, (0.25, 0.35, 0.5), 0.2)
    s1 = scenes.cells_sphere(n, (0.75, 0.35, 0.5), 0.2)
    slab = scenes.cells_slab(n, 3 * dx, 1 - 3 * dx, 3 * dx, 16 * dx, 3 * dx, 1 - 3 * dx)
    assert len(slab) == 250 * 250 * 13
    total = (len(s0) + len(s1) + len(slab)) * 8
    assert abs(total - 15.49e6) / 15.49e6 < 0.005  # ~15.49M particles
