"""Seeded synthetic inputs for the BASELINE.json configurations.

There is no dataset behind this path: BASELINE.json specifies the input
distributions, and these generators reproduce them:

* c1/c2/c3: B ~ N(0,1) i.i.d., columns normalised to unit 2-norm (norms in
  fp64), D = diag(10^(-e*j/(n-1))), A = B*D formed in fp64 then rounded to the
  working precision (e = 6 / 4 / 12);
* c4: A ~ N(0,1) i.i.d. (kappa ~ 1);
* c5: A = U0 diag(sigma) V0^T, sigma_i = 10^(-10(i-1)/(n-1)), U0 the Q factor
  of a Gaussian m x n matrix, V0 Haar n x n (Q of a Gaussian with R's
  diagonal signs absorbed, like proj/src/matgen.cpp:94-108).

Host generation uses numpy's PCG64 (bit-reproducible across platforms);
``device_*`` variants generate on the GPU with torch (used by bench.py for
the multi-GiB configs, where only the distribution matters and the oracle
reads back the stored matrix).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    m: int
    n: int
    working: str  # "f32" | "f64"
    kind: str     # "graded" | "gaussian" | "prescribed"
    decades: float = 0.0


CONFIGS = {
    "c1": Config("c1", 20000, 32, "f32", "graded", 6.0),
    "c2": Config("c2", 1 << 20, 64, "f32", "graded", 4.0),
    "c3": Config("c3", 1 << 22, 256, "f64", "graded", 12.0),
    "c4": Config("c4", 1 << 26, 128, "f32", "gaussian"),
    "c5": Config("c5", 1 << 22, 1024, "f64", "prescribed", 10.0),
}


def graded(m: int, n: int, decades: float, seed: int, dtype=np.float32) -> np.ndarray:
    rng = np.random.default_rng(seed)
    b = rng.standard_normal((n, m))  # row k = column k of B (column-major storage)
    b /= np.sqrt(np.einsum("ij,ij->i", b, b))[:, None]
    d = 10.0 ** (-decades * np.arange(n) / max(n - 1, 1))
    a = (b * d[:, None]).astype(dtype)
    return a.T  # (m, n) Fortran-ordered view


def gaussian(m: int, n: int, seed: int, dtype=np.float32) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.standard_normal((n, m), dtype=np.float64).astype(dtype).T


def haar(n: int, rng) -> np.ndarray:
    q, r = np.linalg.qr(rng.standard_normal((n, n)))
    return q * np.sign(np.diag(r))[None, :]


def prescribed(m: int, n: int, decades: float, seed: int) -> tuple[np.ndarray, np.ndarray]:
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((m, n))
    u0, r = np.linalg.qr(g)
    u0 *= np.sign(np.diag(r))[None, :]
    v0 = haar(n, rng)
    sigma = 10.0 ** (-decades * np.arange(n) / max(n - 1, 1))
    a = np.asfortranarray((u0 * sigma[None, :]) @ v0.T)
    return a, sigma


def make(cfg: Config, seed: int = 1, m: int | None = None):
    """Host matrix for `cfg` (optionally with fewer rows, same distribution)."""
    m = cfg.m if m is None else m
    dt = np.float32 if cfg.working == "f32" else np.float64
    if cfg.kind == "graded":
        return graded(m, cfg.n, cfg.decades, seed, dt)
    if cfg.kind == "gaussian":
        return gaussian(m, cfg.n, seed, dt)
    a, _ = prescribed(m, cfg.n, cfg.decades, seed)
    return a


def device_make(cfg: Config, seed: int = 1, m: int | None = None, device="cuda", rank: int = 0,
                allreduce=None):
    """The same distribution generated on the GPU (torch), column-major as a
    (n, m) row-major tensor whose transpose is the m x n matrix.

    For a row-sharded run each rank passes its ``rank`` (its rows come from
    their own stream) and, for the prescribed-sigma kind, an ``allreduce``
    callable summing an n x n fp64 tensor over ranks, so that U0 is
    orthonormal over the global rows and V0 is shared.
    """
    import torch

    m = cfg.m if m is None else m
    g = torch.Generator(device=device)
    g.manual_seed(seed * 1000003 + rank)
    dt = torch.float32 if cfg.working == "f32" else torch.float64
    n = cfg.n
    if cfg.kind == "gaussian":
        return torch.randn((n, m), generator=g, device=device, dtype=torch.float32).to(dt)
    if cfg.kind == "graded":
        out = torch.empty((n, m), device=device, dtype=dt)
        d = 10.0 ** (-cfg.decades * torch.arange(n, device=device, dtype=torch.float64) / max(n - 1, 1))
        for j in range(n):  # column by column keeps the fp64 scratch at one column
            col = torch.randn(m, generator=g, device=device, dtype=torch.float64)
            col /= torch.linalg.vector_norm(col)
            out[j] = (col * d[j]).to(dt)
        return out
    # prescribed: A^T = V0 diag(sigma) U0^T with U0 from CholQR2 (fp64, on the
    # GPU), kept as U0^T (n x m) throughout so no m x n transpose is needed.
    xt = torch.randn((n, m), generator=g, device=device, dtype=torch.float64)
    for _ in range(2):
        gram = xt @ xt.T
        if allreduce is not None:
            gram = allreduce(gram)
        r = torch.linalg.cholesky(gram, upper=True)
        xt = torch.linalg.solve_triangular(r.T, xt, upper=False, left=True)  # (X R^-1)^T
        del gram, r
    gv_gen = torch.Generator(device=device)
    gv_gen.manual_seed(seed)  # V0 is shared by all ranks
    gv = torch.randn((n, n), generator=gv_gen, device=device, dtype=torch.float64)
    qv, rv = torch.linalg.qr(gv)
    qv = qv * torch.sign(torch.diagonal(rv))[None, :]
    sigma = 10.0 ** (-cfg.decades * torch.arange(n, device=device, dtype=torch.float64) / max(n - 1, 1))
    xt.mul_(sigma[:, None])
    at = qv @ xt
    del xt
    torch.cuda.empty_cache()
    return at
