"""Checks of the synthetic input generator (gen/): exact spectrum, bitwise Hermitian mirroring,
panel consistency (any rank builds any panel bit-identically), thread-count independence, and the
GUE scale (||G||_2 ~ 2)."""
import os
import subprocess
import sys

import numpy as np

import gen as G
from gen.configs import CONFIGS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_spectrum_recipe():
    lam = G.spectrum(512, 480)
    assert lam[0] == -2.0 and abs(lam[479]) < 1e-15 and lam[-1] == 40.0
    assert np.all(np.diff(lam) > 0)
    # density increases toward 0 in the dense part (log-spaced density, R20)
    d = np.diff(lam[:480])
    assert d[0] > d[-1]


def test_h1_exact_and_hermitian():
    w = G.wy(300, 250, 5)
    H = w.full()
    assert np.array_equal(H, H.conj().T)
    assert np.all(np.diag(H).imag == 0)
    np.testing.assert_allclose(np.linalg.eigvalsh(H), w.lam, rtol=0, atol=1e-12 * 40)
    X = w.eigvecs(range(300))
    assert np.abs(X.conj().T @ X - np.eye(300)).max() < 1e-13
    assert np.abs(H @ X - X * w.lam).max() < 1e-12 * 40
    # reflector product: Q = P1...P8 with P_r = I - 2 v v^H / v^H v
    Q = np.eye(300, dtype=complex)
    for r in range(8):
        v = w.V[:, r : r + 1]
        Q = Q @ (np.eye(300) - 2 * (v @ v.conj().T) / np.real(v.conj().T @ v))
    np.testing.assert_allclose(X, Q, atol=1e-13)


def test_panels_match_full():
    w = G.wy(200, 180, 9)
    H = w.full()
    assert np.array_equal(w.panel(37, 50), H[:, 37:87])
    Gf = G.gue(200, 3, G.stream(5, 200))
    assert np.array_equal(G.gue(200, 3, G.stream(5, 200), 120, 80), Gf[:, 120:])
    Y = G.start_basis(200, 6, 4)
    assert np.array_equal(G.start_basis(200, 6, 4, 50, 70), Y[50:120])
    Hp = np.asfortranarray(H[:, 10:30].copy())
    G.perturb(Hp, 1, 2, 0.04, c0=10)
    Hf = H.copy(order="F")
    G.perturb(Hf, 1, 2, 0.04)
    assert np.array_equal(Hp, Hf[:, 10:30])
    assert np.array_equal(Hf, Hf.conj().T)


def test_gue_scale():
    n = 600
    Gm = G.gue(n, 1, G.stream(5, n))
    assert np.array_equal(Gm, Gm.conj().T)
    s = np.linalg.eigvalsh(Gm)
    assert 1.8 < s[-1] < 2.2 and -2.2 < s[0] < -1.8
    assert abs(np.mean(np.abs(Gm) ** 2) * n - 1) < 0.05


def test_thread_count_independence():
    code = ("import numpy as np, gen as G; w = G.wy(257, 200, 3); H = w.panel(0, 257); "
            "import hashlib, sys; sys.stdout.write(hashlib.sha256(H.tobytes()).hexdigest())")
    outs = []
    for t in ("1", "3"):
        env = dict(os.environ, OMP_NUM_THREADS=t, PYTHONPATH=ROOT)
        outs.append(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                                   check=True).stdout)
    assert outs[0] == outs[1]


def test_configs_shapes():
    for name, cf in CONFIGS.items():
        assert cf["nev"] + cf["nex"] <= cf["n"]
        assert cf["n"] % 8 == 0 or name == "c2"  # panels for p = 8 (c2: 13000 = 8 x 1625)
        assert cf["n"] % 8 == 0 or cf["n"] == 13000
