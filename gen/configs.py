"""Workload recipes standing in for the paper's FLEUR sequences (BASELINE.json configs; SURVEY.md
8(d) d2/d3). Pure data: no method arithmetic."""

SEED0 = 1404416100

# name: n, n_d (dense bottom), nev, nex, degree cap, tol, problems in the sequence, delta (perturbation)
CONFIGS = {
    "c0": dict(n=512, nd=480, nev=32, nex=16, cap=20, tol=1e-10, nprob=1, delta=0.0, seed=SEED0 + 0),
    "c1": dict(n=4096, nd=614, nev=200, nex=40, cap=40, tol=1e-10, nprob=5, delta=1e-3, seed=SEED0 + 1),
    "c2": dict(n=13000, nd=1950, nev=520, nex=104, cap=36, tol=1e-10, nprob=10, delta=5e-4, seed=SEED0 + 2),
    "c3": dict(n=30000, nd=4500, nev=1200, nex=240, cap=40, tol=1e-10, nprob=8, delta=2e-4, seed=SEED0 + 3),
}
DEG0 = 8            # R12: starting degree of every problem's first loop
LANCZOS_STEPS = 25  # R17
MAX_LOOPS = 50
HNORM = 40.0        # ||H^(1)||_2 = 40 exactly (R20); the sequence step uses delta * 40 * G_l

# c4 filter-only sweep: H = GUE (stream 5, n), fixed interval
C4_NS = (8192, 16384, 32768)
C4_KS = (64, 256, 1024, 2048)
C4_INTERVAL = dict(lambda1=-2.2, alpha=-1.0, beta=2.2)


def c4_ramp(k: int):
    """Sorted per-vector degrees 8..40: m_j = 8 + round(32 j/(k-1))."""
    if k == 1:
        return [8]
    return [8 + int((32 * j) / (k - 1) + 0.5) for j in range(k)]
