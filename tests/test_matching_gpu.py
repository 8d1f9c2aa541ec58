"""GPU Algorithm 3 (sem_face_match) vs the oracle's literal loop (oracle.matching) on the same seeded
face sets: owners bit-exact, reference coordinates to round-off; full cfg-3-size structured interface
against the closed form of the 2:1 lattice."""
import numpy as np
import pytest

from sem_inputs import interface_faces

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("nfx,nfy,R,N,jitter,seed", [
    (6, 4, 2, 5, 0.0, 0), (6, 6, 3, 3, 0.0, 0), (8, 6, 2, 4, 0.15, 1), (10, 4, 2, 5, 0.2, 2), (6, 6, 3, 2, 0.1, 3)])
def test_matching_parity(nfx, nfy, R, N, jitter, seed):
    from oracle.matching import match_faces
    from paper_2603_06267_b200 import sem_face_match
    fine, coarse = interface_faces(nfx, nfy, R, 25e-6, z0=1e-4, jitter=jitter, seed=seed)
    own_o, xi_o = match_faces(fine, coarse, N)
    own_g, xi_g, ms = sem_face_match(fine, coarse, N)
    assert np.all(own_o >= 0)
    assert np.array_equal(own_g, own_o)
    assert np.max(np.abs(xi_g - xi_o)) < 1e-12


def test_unmatched_node_reported():
    from paper_2603_06267_b200 import sem_face_match
    fine, coarse = interface_faces(4, 4, 2, 25e-6)
    owner, xi, ms = sem_face_match(fine, coarse[:-1], 3)       # drop a coarse face: orphans
    assert np.any(owner < 0) and np.any(owner >= 0)


def test_full_size_structured_closed_form():
    """Config 3's interface lattice (384 x 384 fine faces, N = 5, 2:1): every owner and xhat- equals the
    structured closed form (see tests/test_oracle_matching.py::test_structured_closed_form)."""
    from oracle.gll import gll
    from paper_2603_06267_b200 import sem_face_match
    nf, R, N = 384, 2, 5
    fine, coarse = interface_faces(nf, nf, R, 25e-6, z0=0.6e-3)
    owner, xi, ms = sem_face_match(fine, coarse, N)
    x, _ = gll(N)
    f = np.arange(nf * nf)
    i, j = f % nf, f // nf
    q = np.arange((N + 1) ** 2)
    a, b = q % (N + 1), q // (N + 1)
    I, A = np.meshgrid(i, a, indexing="ij")
    J, B = np.meshgrid(j, b, indexing="ij")

    def axis(I, A):
        e, r, xa = I // R, I % R, x[A]
        edge = (A == 0) & (r == 0) & (e > 0)
        e = np.where(edge, e - 1, e)
        r = np.where(edge, R - 1, r)
        xa = np.where(edge, 1.0, xa)
        return e, (2 * r + xa + 1) / R - 1
    ex, xx = axis(I, A)
    ey, yy = axis(J, B)
    assert np.array_equal(owner, ex + (nf // R) * ey)
    assert np.max(np.abs(xi[..., 0] - xx)) < 1e-12
    assert np.max(np.abs(xi[..., 1] - yy)) < 1e-12
    assert np.max(np.abs(xi[..., 2] + 1)) < 1e-12
