"""The compressed tangent's identities, in fp64 numpy, no GPU: the format k_linearize
writes and k_hvp_wz applies must be the same linear map as K_c : dG = c (C_F : (dG S)) S (S symmetric),
and the Jacobi diagonal's blocks must follow from it.
  * K : dG = U (Chat : (U^T dG W)) W^T with W = S V (so no separate S in the HVP);
  * flipping a column pair of U and V (U D, V D, det D = 1) leaves that map unchanged, and choosing the
    pair that moves U's largest quaternion component into w gives |w| >= 1/2, so (x, y, z) in fp32
    recover U to ~1e-7;
  * K[(a,b),(a,e)] = X_b : Chat : X_e with X_b = u_a w_b^T (u_a = row a of U, w_b = row b of W)."""
import numpy as np

PAIRS = [(0, 1), (0, 2), (1, 2)]


def _rot(rng):
    q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    if np.linalg.det(q) < 0:
        q[:, 0] *= -1
    return q


def _chat(psi, ab, X):
    Y = np.zeros((3, 3))
    for i in range(3):
        Y[i, i] = psi[i] @ np.diag(X)
    for p, (i, j) in enumerate(PAIRS):
        a, b = ab[p]
        Y[i, j], Y[j, i] = a * X[i, j] + b * X[j, i], b * X[i, j] + a * X[j, i]
    return Y


def _case(seed):
    rng = np.random.default_rng(seed)
    U, V = _rot(rng), _rot(rng)
    S = np.eye(3) + 0.2 * rng.normal(size=(3, 3))
    S = 0.5 * (S + S.T)
    psi = rng.normal(size=(3, 3))
    return U, V, S, psi + psi.T, rng.normal(size=(3, 2))


def _matrix(apply):
    M = np.zeros((9, 9))
    for c in range(9):
        E = np.zeros((3, 3))
        E.flat[c] = 1.0
        M[:, c] = apply(E).ravel()
    return M


def _quat(R):  # Shepperd, as k_linearize's rot_quat
    t = np.trace(R)
    if t > 0:
        s = 2 * np.sqrt(t + 1)
        q = [0.25 * s, (R[2, 1] - R[1, 2]) / s, (R[0, 2] - R[2, 0]) / s, (R[1, 0] - R[0, 1]) / s]
    elif R[0, 0] > R[1, 1] and R[0, 0] > R[2, 2]:
        s = 2 * np.sqrt(1 + R[0, 0] - R[1, 1] - R[2, 2])
        q = [(R[2, 1] - R[1, 2]) / s, 0.25 * s, (R[0, 1] + R[1, 0]) / s, (R[0, 2] + R[2, 0]) / s]
    elif R[1, 1] > R[2, 2]:
        s = 2 * np.sqrt(1 + R[1, 1] - R[0, 0] - R[2, 2])
        q = [(R[0, 2] - R[2, 0]) / s, (R[0, 1] + R[1, 0]) / s, 0.25 * s, (R[1, 2] + R[2, 1]) / s]
    else:
        s = 2 * np.sqrt(1 + R[2, 2] - R[0, 0] - R[1, 1])
        q = [(R[1, 0] - R[0, 1]) / s, (R[0, 2] + R[2, 0]) / s, (R[1, 2] + R[2, 1]) / s, 0.25 * s]
    q = np.array(q)
    return q / np.linalg.norm(q)


def _quat_rot(w, x, y, z):
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def test_w_form_is_the_tangent():
    for seed in range(20):
        U, V, S, psi, ab = _case(seed)
        ref = _matrix(lambda dG: U @ _chat(psi, ab, U.T @ (dG @ S) @ V) @ V.T @ S)
        W = S @ V
        got = _matrix(lambda dG: U @ _chat(psi, ab, U.T @ dG @ W) @ W.T)
        assert np.allclose(got, ref, rtol=0, atol=1e-12)
        assert np.allclose(ref, ref.T, atol=1e-12)  # a symmetric tangent


def test_column_pair_flip_and_three_component_quaternion():
    worst = 0.0
    for seed in range(2000):
        U, V, S, psi, ab = _case(seed)
        W = S @ V
        ref = _matrix(lambda dG: U @ _chat(psi, ab, U.T @ dG @ W) @ W.T)
        q = _quat(U)
        m = int(np.argmax(np.abs(q)))
        if m:
            D = np.array([1.0 if m == 1 else -1.0, 1.0 if m == 2 else -1.0, 1.0 if m == 3 else -1.0])
            U, W = U * D, W * D
            q = _quat(U)
        q = q if q[0] >= 0 else -q
        assert q[0] >= 0.5 - 1e-12
        got = _matrix(lambda dG: U @ _chat(psi, ab, U.T @ dG @ W) @ W.T)
        assert np.allclose(got, ref, rtol=0, atol=1e-12)
        x, y, z = (float(np.float32(c)) for c in q[1:])
        w = np.sqrt(1.0 - (x * x + y * y + z * z))
        worst = max(worst, np.abs(_quat_rot(w, x, y, z) - U).max())
    assert worst < 1e-6


def test_diagonal_blocks_from_the_compressed_form():
    for seed in range(20):
        U, V, S, psi, ab = _case(seed)
        W = S @ V
        M = _matrix(lambda dG: U @ _chat(psi, ab, U.T @ dG @ W) @ W.T)
        for a in range(3):
            X = [np.outer(U[a], W[b]) for b in range(3)]
            for b in range(3):
                for e in range(3):
                    val = np.sum(X[b] * _chat(psi, ab, X[e]))
                    assert abs(val - M[3 * a + b, 3 * a + e]) < 1e-12
