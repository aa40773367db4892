"""Interior grid of the unit square (mirror of `pkg/src/ocp/grid.py:9-91`).

Same indexing contract as the reference: ``n`` interior points per
dimension, ``h = 1/(n+1)``, flat row-major index ``k = i*n + j`` for the point
``((i+1)h, (j+1)h)`` (`grid.py:26-61`).  The device path never materialises
the Laplacian: its kernels apply the 5-point stencil with the coefficients
``4/h^2`` and ``-1/h^2`` of `build_laplacian` (`grid.py:83-91`).  The sparse
matrix is still built here for callers that hand a ``ProblemSpec.a`` around.
"""

from dataclasses import dataclass

import numpy as np


class NonfiniteFieldError(ValueError):
    """A field operation produced a NaN or Inf entry (`grid.py:9-15`)."""

    def __init__(self, where, index):
        self.where = where
        self.index = index
        super().__init__(f"nonfinite value in {where} at flat index {index}")


def check_finite(v, where):
    """Return v, raising NonfiniteFieldError at the first bad entry (`grid.py:18-23`)."""
    bad = ~np.isfinite(v)
    if bad.any():
        raise NonfiniteFieldError(where, int(np.argmax(bad)))
    return v


@dataclass(frozen=True)
class Grid:
    n: int

    def __post_init__(self):
        if self.n < 1:
            raise ValueError("grid needs at least one interior point per dimension")

    @property
    def h(self):
        return 1.0 / (self.n + 1)

    @property
    def size(self):
        return self.n * self.n

    def index(self, i, j):
        return i * self.n + j

    def coords(self, k):
        return divmod(int(k), self.n)

    def points(self):
        t = self.h * np.arange(1, self.n + 1)
        x1 = np.repeat(t, self.n)
        x2 = np.tile(t, self.n)
        return x1, x2

    def inner(self, u, v):
        return self.h ** 2 * float(np.dot(u, v))

    def norm(self, u):
        return float(np.sqrt(self.inner(u, u)))


def build_laplacian(grid):
    """Sparse 5-point -Laplacian / h^2 with Dirichlet rows eliminated.

    Host-side convenience only (ProblemSpec compatibility); entries are
    exactly the reference's: 4/h^2 on the diagonal, -1/h^2 to the four
    neighbours, column indices sorted within each row.
    """
    import scipy.sparse as sp

    n = grid.n
    h2 = grid.h ** 2
    k = np.arange(n * n)
    i, j = np.divmod(k, n)
    rows, cols, vals = [k], [k], [np.full(n * n, 4.0 / h2)]
    for di, dj in ((-1, 0), (0, -1), (0, 1), (1, 0)):
        ii, jj = i + di, j + dj
        m = (ii >= 0) & (ii < n) & (jj >= 0) & (jj < n)
        rows.append(k[m])
        cols.append(ii[m] * n + jj[m])
        vals.append(np.full(int(m.sum()), -1.0 / h2))
    a = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n * n, n * n))
    a.sort_indices()
    return a
