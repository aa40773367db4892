"""Full-grid parity checks of a solve against a reference-made fixture.

The north-star bar (BASELINE.json): y, p, u within 1e-8 relative L2 of the
reference, and an identical control support {u != 0} except where |p| lies
within eps of the threshold mu.

Fixtures up to 256^2 hold the full vectors.  Larger ones (configs 3 and 4)
hold, per field, a digest of the FULL vector made by
``tests/golden/make_golden.py digest``:

* ``*_proj``: P projections s_k . v with seeded random signs s_k in {-1, +1}^N.
  For a difference e = v_gpu - v_ref, E[(s_k . e)^2] = ||e||^2, so
  sqrt(mean_k (s_k . v_gpu - proj_k)^2) estimates ||e||_2 over the whole
  vector (P = 16: the estimate falls below half the true error with
  probability < 1e-3).  The test bounds that estimate by 1e-8 ||v_ref||.
* ``*_samples`` / ``*_norm``: a strided sample and the norm.
* ``supp_bits`` / ``band_bits``: bit-packed |p| > mu and ||p| - mu| <= eps
  of the reference's p over every grid point, so the support criterion is
  checked on the whole grid.
"""

import numpy as np

DIGEST_SEED = 20241101   # tests/golden/make_golden.py
REL_L2 = 1e-8


def rel_l2(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def signs(n, rows):
    rng = np.random.default_rng(DIGEST_SEED + n)
    return rng.integers(0, 2, size=(rows, n)).astype(np.float64) * 2.0 - 1.0


def projected_error(vec, proj, s):
    """Estimate of ||vec - v_ref||_2 from the reference's projections."""
    return float(np.sqrt(np.mean((s @ vec - proj) ** 2)))


def check_fields(g, fields, mu, eps, tol=REL_L2):
    """Assert the BASELINE parity bar for ``fields`` = {"y": y, "p": p, "u": u}."""
    p = fields["p"]
    n2 = p.shape[0]
    if "y" in g.files:
        for key, vec in fields.items():
            assert rel_l2(vec, g[key]) <= tol, (key, rel_l2(vec, g[key]))
        p_ref = g["p"]
        support_ref = np.abs(p_ref) > mu
        band = np.abs(np.abs(p_ref) - mu) <= eps
    else:
        s = None
        for key, vec in fields.items():
            stride = int(g[f"{key}_stride"])
            assert rel_l2(vec[::stride], g[f"{key}_samples"]) <= tol, key
            ref_norm = float(g[f"{key}_norm"])
            assert abs(np.linalg.norm(vec) - ref_norm) <= tol * ref_norm, key
            proj = g[f"{key}_proj"]
            if s is None:
                s = signs(n2, proj.shape[0])
            err = projected_error(vec, proj, s)
            assert err <= tol * ref_norm, (key, err / ref_norm)
        assert "supp_bits" in g.files, "fixture lacks the full-grid support bitmap"
        support_ref = np.unpackbits(g["supp_bits"])[:n2].astype(bool)
        band = np.unpackbits(g["band_bits"])[:n2].astype(bool)
        assert int(g["supp_count"]) == int(support_ref.sum())
    support = np.abs(p) > mu
    mism = np.flatnonzero((support != support_ref) & ~band)
    assert mism.size == 0, f"control support differs at {mism.size} points outside the band"
    return int(support_ref.sum()), int(band.sum())
