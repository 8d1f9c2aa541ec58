"""Pins of the oracle's rigid obstacles: solid elements are removed from the
fluid, so the faces they share with fluid elements are Neumann surfaces -- the natural boundary
condition of the weak form (Eq. 4 has no boundary term there).  Pinned against what that
fixes independently of the obstacle code path:
  * a solid top layer is the same problem as the box without that layer and a rigid top face
    (also with an absorbing side face, whose solid-layer part must then not absorb);
  * a solid wall splits the box into two fluids that share no node: a field started on one side
    never reaches the other (exact zeros), and each side equals the box cut at the wall;
  * a curved box with an obstacle keeps the discrete energy of a closed rigid cavity bounded.
"""
import numpy as np

from oracle.newmark import Newmark
from oracle.operators import System
from sem_inputs import BC_ABSORBING, BC_RIGID, obstacle_config, solid_block


def _run(rec, p0, v0, n):
    nm = Newmark(System(rec))
    nm.set_state(p0, v0)
    nm.run(n)
    return nm


def _grid(nel, N):
    return tuple(N * e + 1 for e in nel)


def _embed(small, nel_small, nel_big, N):
    """Values on the small box lattice placed into the big box lattice (same origin, same h)."""
    ns, nb = _grid(nel_small, N), _grid(nel_big, N)
    out = np.zeros(nb[0] * nb[1] * nb[2])
    s = small.reshape(ns[2], ns[1], ns[0])
    o = out.reshape(nb[2], nb[1], nb[0])
    o[:ns[2], :ns[1], :ns[0]] = s
    return out


def _restrict(big, nel_small, nel_big, N):
    ns, nb = _grid(nel_small, N), _grid(nel_big, N)
    return big.reshape(nb[2], nb[1], nb[0])[:ns[2], :ns[1], :ns[0]].ravel()


def _field(n, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(n), 1e7 * rng.standard_normal(n)


def test_solid_top_layer_equals_rigid_top_face():
    N, nel_big, nel_small = 3, (3, 2, 4), (3, 2, 3)
    for bc in ([BC_RIGID] * 6, [BC_RIGID, BC_ABSORBING] + [BC_RIGID] * 4):
        big = obstacle_config(nel=nel_big, degree=N, solid_lo=(0, 0, 3), solid_hi=(3, 2, 4), bc=bc)
        small = obstacle_config(nel=nel_small, degree=N, solid_lo=(0, 0, 0), solid_hi=(0, 0, 0), bc=bc)
        small["dt"] = big["dt"]
        ns = np.prod(_grid(nel_small, N))
        p0, v0 = _field(ns, 3)
        a = _run(big, _embed(p0, nel_small, nel_big, N), _embed(v0, nel_small, nel_big, N), 40)
        b = _run(small, p0, v0, 40)
        pa = _restrict(a.p, nel_small, nel_big, N)
        assert np.max(np.abs(pa - b.p)) <= 1e-12 * np.max(np.abs(b.p)), bc
        # nodes above the shared plane belong to no fluid element: 0
        nb = _grid(nel_big, N)
        above = a.p.reshape(nb[2], nb[1], nb[0])[N * 3 + 1:]
        assert np.all(above == 0.0)


def test_solid_wall_decouples_the_two_fluids():
    N, nel = 3, (7, 2, 2)
    rec = obstacle_config(nel=nel, degree=N, solid_lo=(3, 0, 0), solid_hi=(4, 2, 2), bc=[BC_RIGID] * 6)
    nn = _grid(nel, N)
    gx = np.tile(np.arange(nn[0]), nn[1] * nn[2])
    left = gx <= 3 * N
    right = gx >= 4 * N
    p0, v0 = _field(len(gx), 5)
    p0[~left] = 0.0
    v0[~left] = 0.0
    nm = _run(rec, p0, v0, 60)
    assert np.all(nm.p[right] == 0.0) and np.all(nm.pd[right] == 0.0)
    assert np.max(np.abs(nm.p[left])) > 0.1
    # the left fluid alone is the box cut at the wall with a rigid +x face
    small = obstacle_config(nel=(3, 2, 2), degree=N, solid_lo=(0, 0, 0), solid_hi=(0, 0, 0), bc=[BC_RIGID] * 6)
    small["dt"] = rec["dt"]
    ns = _grid((3, 2, 2), N)
    sel = left.reshape(nn[2], nn[1], nn[0])
    ps = p0.reshape(nn[2], nn[1], nn[0])[sel].reshape(ns[2], ns[1], ns[0]).ravel()
    vs = v0.reshape(nn[2], nn[1], nn[0])[sel].reshape(ns[2], ns[1], ns[0]).ravel()
    b = _run(small, ps, vs, 60)
    pl = nm.p.reshape(nn[2], nn[1], nn[0])[sel]
    assert np.max(np.abs(pl - b.p)) <= 1e-12 * np.max(np.abs(b.p))


def test_curved_obstacle_energy_bounded_and_interior_zero():
    rec = obstacle_config(nel=(4, 4, 3), degree=3, solid_lo=(1, 1, 1), solid_hi=(3, 3, 2),
                          bc=[BC_RIGID] * 6, curved_amp=0.12, seed=4)
    s = System(rec)
    n = s.ndof
    p0, v0 = _field(n, 9)
    nm = Newmark(s)
    nm.set_state(p0, v0)
    nm.step()
    e0 = nm.energy()
    es = []
    for _ in range(200):
        nm.step()
        es.append(nm.energy())
    # explicit central differences conserve a modified energy: the plain one oscillates within a few %
    assert max(abs(e / e0 - 1.0) for e in es) < 0.05
    assert np.all(nm.p[~s.active] == 0.0)
    # the obstacle has interior nodes (the 2 x 2 x 1 solid block of N = 3 elements: 5 x 5 x 2 ... minus
    # its surface) -- here the block's interior lattice points (gx, gy in N+1..3N-1, gz in N+1..2N-1)
    assert (~s.active).sum() == (2 * 3 - 1) ** 2 * (3 - 1)


def test_solid_block_indices():
    idx = solid_block((4, 3, 2), (1, 0, 1), (3, 2, 2))
    ex, ey, ez = idx % 4, (idx // 4) % 3, idx // 12
    assert len(idx) == 4 and np.all((ex >= 1) & (ex < 3) & (ey < 2) & (ez == 1))
