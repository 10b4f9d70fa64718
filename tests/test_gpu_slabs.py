"""GPU parity of the slab decomposition on ONE GPU.

R slab ranks run as host threads of this process through the library's in-process loopback group
(mpl_group_create): every collective synchronises the rank's stream and meets the other ranks at a host
barrier, so no kernel ever waits on another rank's kernel (B200_PROFILING.md: ranks must not spin on
each other on one GPU).  The NCCL transport runs the same code with ncclAllReduce / ncclSend / ncclRecv
in place of the barrier + copy.

Checks, against the fp64 oracle on the same seeded scene: the union of the owned active blocks and
owned nodes is bit-exact; energies agree on every rank; gradient / HVP / Jacobi diagonal on owned nodes
and the replayed full step (v^{n+1} and particle state gathered by global id) meet the single-GPU bars;
copies of shared interface nodes are bitwise equal on the two ranks that hold them.  A multi-step run
with particles crossing the cuts (migration + ghost refresh) matches the single-rank GPU run."""
import concurrent.futures as cf
import dataclasses

import numpy as np
import pytest

import oracle
from paper_2602_07853_b200 import mpl, scenes

from ._parity import TOL, node_ids, rel_l2
from .test_gpu_parity import small_cfg2, two_material

pytestmark = pytest.mark.gpu


def run_ranks(R, fn):
    with cf.ThreadPoolExecutor(R) as ex:
        futs = [ex.submit(fn, r) for r in range(R)]
        return [f.result(timeout=900) for f in futs]


def _q(sc):
    dt_ = sc.dtype
    return dataclasses.replace(sc, x=sc.x.astype(dt_), v=sc.v.astype(dt_), F=sc.F.astype(dt_), G=sc.G.astype(dt_),
                               vol=sc.vol.astype(dt_))


CASES = {
    "cfg1_R2": (lambda: scenes.cfg1(prestrain=True), [0, 2, 4]),
    "cfg2s_fp32_R3": (lambda: small_cfg2(32), [0, 3, 4, 8]),
    "cfg2s_fp64_R4": (lambda: small_cfg2(64), [0, 3, 4, 5, 8]),
    # one 4-cell block plane per rank; ranks 0, 1, 6, 7 hold no cells (only ghost / empty slabs)
    "cfg2s_fp32_R8": (lambda: small_cfg2(32), [0, 1, 2, 3, 4, 5, 6, 7, 8]),
    "mix_fp64_R2": (lambda: two_material(64), [0, 2, 4]),
    "lawmix_fp32_R2": (lambda: two_material(32, (1, 0)), [0, 2, 4]),  # split Neo-Hookean + Hencky
    "watermix_fp64_R2": (lambda: two_material(64, (0, 2)), [0, 2, 4]),  # Hencky + J-based water
    "vmmix_fp64_R2": (lambda: two_material(64, (0, 0), (1500.0, 0.0)), [0, 2, 4]),  # von Mises + elastic
}


class SlabRun:
    def __init__(self, sc, cuts):
        self.sc = sc
        self.cuts = np.asarray(cuts, np.int32)
        self.R = len(cuts) - 1
        self.grid = oracle.Grid(sc.n, sc.dx, sc.origin)
        self.un, self.S, self.prob, self.v0 = oracle.prepare(sc, self.grid)
        rng = np.random.default_rng(5)
        act = (self.un.m_i > 0)[:, None]
        self.vp = self.v0 + 0.01 * rng.normal(size=self.v0.shape) * act
        self.u = np.random.default_rng(4).normal(size=self.v0.shape) * act
        if sc.precision == 32:
            self.vp = self.vp.astype(np.float32).astype(np.float64)
            self.u = self.u.astype(np.float32).astype(np.float64)
        st_o = self.prob.newton(self.v0, sc.solver)[1]
        self.counts_o = st_o
        self.v_o, _ = self.prob.newton(self.v0, sc.solver, st_o["newton_iters"], st_o["cg_iters"], st_o["ls_iters"])
        self.group = mpl.Group(self.R)
        self.res = run_ranks(self.R, self.rank_fn)
        self.group.close()

    def rank_fn(self, r):
        sc = self.sc
        ctx = mpl.from_scene_rank(sc, r, self.R, self.cuts, device=0, group=self.group)
        try:
            ctx.resample(sc.dt)
            out = {}
            out["blocks"] = ctx.get_active_blocks()
            ijk, m, vn, free = ctx.get_nodes()
            nid = node_ids(self.grid, ijk)
            out.update(nid=nid, m=m, vn=vn, free=free, own=ctx.get_node_owner())
            dt_ = ctx.dtype
            vp = np.ascontiguousarray(self.vp[nid], dt_)
            g, phi = ctx.gradient(vp)
            out.update(g=g, phi=phi, e=ctx.energy(vp))
            ctx.linearize(vp)
            out["h"] = ctx.hvp(np.ascontiguousarray(self.u[nid], dt_))
            out["D"] = ctx.get_diag()
            ctx.set_velocity(np.ascontiguousarray(self.v0[nid], dt_))
            c = self.counts_o
            out["st"] = ctx.newton_step(sc.solver, c["newton_iters"], c["cg_iters"], c["ls_iters"])
            out["v"] = ctx.get_velocity()
            ctx.transfer_to_particles(sc.dt)
            out["ids"] = ctx.get_particle_ids()
            out["x"], out["pv"], out["F"], out["G"] = ctx.get_particles()
            return out
        finally:
            ctx.close()

    def owned(self, key):
        nid = np.concatenate([o["nid"][o["own"] == 1] for o in self.res])
        val = np.concatenate([o[key][o["own"] == 1] for o in self.res])
        return nid, val


@pytest.fixture(scope="module", params=list(CASES))
def run(request):
    mk, cuts = CASES[request.param]
    return SlabRun(_q(mk()), cuts)


def test_owned_blocks_and_nodes_partition(run):
    base = oracle.base_cells(run.grid, run.sc.x)
    blocks = np.concatenate([o["blocks"] for o in run.res])
    assert np.array_equal(np.sort(blocks), oracle.active_blocks(run.grid, base))
    nid, _ = run.owned("m")
    assert len(nid) == len(np.unique(nid)), "a node is owned by two ranks"
    assert set(nid.tolist()) == set(np.nonzero(run.un.m_i > 0)[0].tolist())
    # every rank holds only the nodes of its slab (plus the shared plane)
    for r, o in enumerate(run.res):
        ix = o["nid"] // ((run.grid.n[1] + 1) * (run.grid.n[2] + 1))
        if len(ix) == 0:  # a slab without active nodes (R8: the outer block planes)
            continue
        assert ix.min() >= 4 * run.cuts[r] and ix.max() <= 4 * run.cuts[r + 1]


def test_unload_on_owned_nodes(run):
    tol = TOL[run.sc.precision]["unload"]
    nid, m = run.owned("m")
    assert rel_l2(m, run.un.m_i[nid]) <= tol
    nid, vn = run.owned("vn")
    assert rel_l2(vn, run.un.v_i[nid]) <= tol
    nid, fr = run.owned("free")
    assert np.array_equal(fr.astype(bool), run.prob.freed[nid] != 0)


def test_energy_gradient_hvp_diag(run):
    tol = TOL[run.sc.precision]
    po = run.prob
    if any(getattr(m, "yield_stress", 0.0) > 0 for m in run.sc.materials):  # bases re-projected at vp
        po = run.prob.with_bases(run.prob.plastic_update(run.vp)[0])
    phi_o = po.energy(run.vp)
    for o in run.res:  # the energy is global: every rank reports it
        assert abs(o["phi"] - phi_o) <= tol["grad"] * abs(phi_o)
        assert abs(o["e"] - phi_o) <= tol["grad"] * abs(phi_o)
    nid, g = run.owned("g")
    assert rel_l2(g, po.gradient(run.vp)[nid]) <= tol["grad"]
    nid, h = run.owned("h")
    assert rel_l2(h, po.hvp(run.vp, run.u)[nid]) <= tol["hvp"]
    nid, D = run.owned("D")
    assert rel_l2(D, po.diag(run.vp)[nid]) <= tol["hvp"]


def test_shared_nodes_bitwise_consistent(run):
    """Both copies of an interface node carry identical gradient, HVP and v^{n+1}."""
    shared = 0
    for r in range(run.R - 1):
        a, b = run.res[r], run.res[r + 1]
        # neighbours share the active nodes of their cut's node plane (none when a slab is empty)
        common, ia, ib = np.intersect1d(a["nid"], b["nid"], return_indices=True)
        shared += len(common)
        for key in ("m", "g", "h", "D", "v"):
            assert np.array_equal(a[key][ia], b[key][ib]), key
        assert np.all(a["own"][ia] + b["own"][ib] == 1)
    assert shared > 0


def test_replayed_step(run):
    sc = run.sc
    tol = TOL[sc.precision]["step"]
    for o in run.res:
        assert o["st"]["newton_iters"] == run.counts_o["newton_iters"]
        assert o["st"]["cg_iters"] == run.counts_o["cg_iters"]
    nid, v = run.owned("v")
    assert rel_l2(v, run.v_o[nid]) <= tol
    ids = np.concatenate([o["ids"] for o in run.res])
    assert np.array_equal(np.sort(ids), np.arange(sc.n_particles))
    order = np.argsort(ids)
    x_o, vp_o, F_o, G_o = oracle.g2p(run.grid, sc.dt, run.un.m_c, run.v_o, sc.x, sc.v, sc.F, sc.G, mat=sc.mat,
                                     materials=sc.materials)
    for key, ref, t in (("x", x_o, tol), ("pv", vp_o, tol), ("F", F_o, tol), ("G", G_o, tol * 10)):
        got = np.concatenate([o[key] for o in run.res])[order]
        assert rel_l2(got, ref) <= t, key


def test_migration_multistep_matches_one_rank():
    """Particles translate across the cuts (about 0.3 cells per step): migration and the ghost layer
    are refreshed every step; five adaptive steps agree with the single-rank GPU run."""
    sc = scenes.cfg1(prestrain=True)
    sc = dataclasses.replace(sc, v=sc.v + np.array([20.0, 0.0, 0.0]))
    steps = 5
    one = mpl.from_scene(sc, 0)
    for _ in range(steps):
        one.step(sc.dt, sc.solver)
    x1, v1, F1, G1 = one.get_particles()
    one.close()
    cuts = np.array([0, 2, 4], np.int32)
    R = 2
    grp = mpl.Group(R)

    def fn(r):
        ctx = mpl.from_scene_rank(sc, r, R, cuts, device=0, group=grp)
        n0 = ctx.num_particles()
        try:
            for _ in range(steps):
                ctx.step(sc.dt, sc.solver)
            return n0, ctx.get_particle_ids(), ctx.get_particles()
        finally:
            ctx.close()

    res = run_ranks(R, fn)
    grp.close()
    ids = np.concatenate([r[1] for r in res])
    assert np.array_equal(np.sort(ids), np.arange(sc.n_particles))
    moved = sum(abs(len(r[1]) - r[0]) for r in res)
    assert moved > 0, "no particle crossed a cut: the migration path was not exercised"
    order = np.argsort(ids)
    for k, ref in enumerate((x1, v1, F1, G1)):
        got = np.concatenate([r[2][k] for r in res])[order]
        assert rel_l2(got, ref) <= 1e-7, k


def test_migration_multistep_eight_ranks():
    """The 32^3 cfg2 block moving +x at about 0.3 cells per step over 8 one-plane slabs (four of them
    start empty): particles migrate into empty ranks; five adaptive steps agree with one rank."""
    sc = small_cfg2(64)
    sc = dataclasses.replace(sc, v=sc.v + np.array([5.0, 0.0, 0.0]))
    steps = 5
    one = mpl.from_scene(sc, 0)
    for _ in range(steps):
        one.step(sc.dt, sc.solver)
    x1, v1, F1, G1 = one.get_particles()
    one.close()
    R = 8
    cuts = np.arange(R + 1, dtype=np.int32)
    grp = mpl.Group(R)

    def fn(r):
        ctx = mpl.from_scene_rank(sc, r, R, cuts, device=0, group=grp)
        n0 = ctx.num_particles()
        try:
            for _ in range(steps):
                ctx.step(sc.dt, sc.solver)
            return n0, ctx.get_particle_ids(), ctx.get_particles()
        finally:
            ctx.close()

    res = run_ranks(R, fn)
    grp.close()
    ids = np.concatenate([r[1] for r in res])
    assert np.array_equal(np.sort(ids), np.arange(sc.n_particles))
    assert sum(abs(len(r[1]) - r[0]) for r in res) > 0
    order = np.argsort(ids)
    for k, ref in enumerate((x1, v1, F1, G1)):
        got = np.concatenate([r[2][k] for r in res])[order]
        assert rel_l2(got, ref) <= 1e-7, k


def test_collective_error_reaches_every_rank():
    """A particle outside the grid on one rank fails the resample on every rank (no hang)."""
    sc = scenes.cfg1()
    cuts = np.array([0, 2, 4], np.int32)
    grp = mpl.Group(2)

    def fn(r):
        ctx = mpl.from_scene_rank(sc, r, 2, cuts, device=0, group=grp)
        try:
            if r == 1:
                x = sc.x[mpl.slab_select(sc, cuts, 1)].copy()
                x[0, 1] = 0.999  # base cell N-1: stencil leaves the grid
                sel = mpl.slab_select(sc, cuts, 1)
                ctx.set_particles(x, sc.v[sel], sc.F[sel], sc.G[sel], sc.vol[sel], sc.mat[sel])
                ctx.set_particle_ids(sel.astype(np.int32))
            try:
                ctx.resample(sc.dt)
                return None
            except mpl.MplError as e:
                return e.code
        finally:
            ctx.close()

    codes = run_ranks(2, fn)
    grp.close()
    assert codes[1] == 3  # MPL_ERR_OUT_OF_DOMAIN where it happened
    assert codes[0] is not None  # and an error (not a hang) on the other rank


def test_nccl_transport_selftest():
    """The NCCL entry points the slab transport uses work on this GPU (one-rank communicator)."""
    import torch  # noqa: F401  (loads torch's NCCL first, as bench.py does)
    assert mpl.nccl_selftest(0) == 8.0
    uid = mpl.nccl_unique_id()
    assert len(uid) == 128
