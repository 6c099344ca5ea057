"""Oracle checks of converged eigenproblems whose spectrum is not known in closed form (the perturbed
problems of a sequence): shared by the GPU parity tests. Test infrastructure: calls only oracle/."""
import oracle as O


def check_perturbed(H, lam, X, nev, tol, seed, inertia):
    """Oracle checks of one converged eigenproblem of a perturbed sequence (SURVEY 8(c) c4 rows (ii) and
    (iii); Alg 1 "Ensure" and locking), all in the oracle's naive loops:
      (i)  residuals ||H x - lam x|| / ||H|| <= tol on 9 sampled eigenvectors (0..2, the middle three,
           nev-3..nev-1), normalised by a certified LOWER bound of ||H||_2: the largest |Ritz value| of the
           oracle's Lanczos tridiagonal (Ritz values are Rayleigh quotients, so |theta| <= ||H||_2);
      (ii) the Kato-Temple bound r^2 / gap (<= 1e-12 |rho| asserted) on the distance from the oracle's
           Rayleigh quotient rho of the GPU's vector to the eigenvalue it approximates, the gap taken from
           the neighbouring Rayleigh quotients minus their residuals (for nev-1 the neighbour above is the
           first buffer vector); with |lam_gpu - rho| it bounds the GPU eigenvalue's error by 1e-10 |rho| (J);
      (iii) completeness ("the nev smallest"): Sylvester inertia of H - sigma I (Bunch-Kaufman) with sigma
           just above the largest wanted eigenvalue counts exactly nev eigenvalues below."""
    m = nev // 2
    windows = [list(range(0, 4)), list(range(m - 2, m + 3)), list(range(nev - 4, nev + 1))]
    cols = sorted({j for w in windows for j in w})
    rho, ra = O.rayleigh_quotients(H, X[:, cols])
    R = dict(zip(cols, zip(rho, ra)))
    tmin, tmax, _ = O.lanczos(H, 25, seed)
    h_lo = max(abs(tmin), abs(tmax))
    sample = [0, 1, 2, m - 1, m, m + 1, nev - 3, nev - 2, nev - 1]
    res = O.residuals(H, X[:, sample], lam[sample], h_lo)  # (i)
    assert res.max() <= tol, res
    for j in sample:  # (ii): |lam_gpu - lam_true| <= |lam_gpu - rho| + r^2 / gap <= 1e-10 |rho| (J)
        r, rj = R[j]
        gaps = [abs(R[i][0] - r) - R[i][1] for i in (j - 1, j + 1) if i in R]
        gap = min(gaps)
        assert gap > 0, (j, gaps)
        assert rj * rj / gap <= 1e-12 * abs(r), (j, rj, gap)
        assert abs(lam[j] - r) + rj * rj / gap <= 1e-10 * abs(r), (j, lam[j], r, rj, gap)
    if inertia:  # (iii)
        sigma = lam[nev - 1] + min(1e-6, 0.5 * (R[nev][0] - lam[nev - 1]))
        assert O.count_below(H, sigma) == nev
