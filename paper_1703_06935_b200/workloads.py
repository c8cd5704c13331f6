"""Seeded synthetic stand-ins for the BASELINE.json configurations C1..C5.

The paper measures on Oxford/Paris/Instre CNN descriptors (reference
``PAPER.md:269-276``); none of those datasets exist here, so each BASELINE
config is replaced by Gaussian clusters with the config's shapes
(SURVEY.md section 8(d)).  Everything is drawn from ONE
``numpy.random.default_rng(seed)`` in a fixed order -- centres, labels,
noise, held-out queries -- so the same seed gives the same data on every host.

C3/C4 do not fit a host-side numpy pipeline (n*d*8 bytes = 16 GB at C3), so
``device_cluster_descriptors`` generates them on the GPU with a seeded torch
generator instead.  There is no CPU parity at those sizes;
what matters there is shape, sparsity and value distribution.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    seed: int
    n: int
    d: int
    clusters: int
    sigma: float
    zipf: float | None
    k: int            # mutual-kNN neighbours
    gamma: float
    r: int
    p: int
    q: int
    density: float    # tau = round(density * n * r)
    queries: int
    y_top: int        # nonzeros kept per observation vector
    alpha: float = 0.99

    @property
    def r_hat(self) -> int:
        return min(self.r + self.p, self.n)

    @property
    def tau(self) -> int:
        return int(round(self.density * self.n * self.r))


@dataclass(frozen=True)
class RegionalConfig:
    """BASELINE C4: ``images`` images x ``regions`` region descriptors (the
    regions of one image = its centre + sigma noise), n = images * regions;
    a query is a re-photographed database image: its ``regions`` regions
    pooled into one observation vector (ranking.py:190-216)."""

    name: str
    seed: int
    images: int
    regions: int
    d: int
    sigma: float
    k: int
    gamma: float
    r: int
    p: int
    q: int
    density: float
    queries: int
    y_top: int
    alpha: float = 0.99

    @property
    def n(self) -> int:
        return self.images * self.regions

    @property
    def r_hat(self) -> int:
        return min(self.r + self.p, self.n)

    @property
    def tau(self) -> int:
        return int(round(self.density * self.n * self.r))


# C4 at full size needs the 8-GPU sharded path (n x r_hat fp32 = 110 GB per block);
# C4r is its generator at 4000 images (n = 20k) for parity against the reference.
REGIONAL = {
    "C4": RegionalConfig("C4", 4, 500_000, 5, 512, 0.05, 50, 3.0, 10_000, 1_000, 3, 0.02, 1_000, 50),
    "C4r": RegionalConfig("C4r", 4, 4_000, 5, 512, 0.05, 50, 3.0, 400, 40, 3, 0.02, 30, 50),
}


def regional_descriptors(cfg: RegionalConfig):
    """(data (n x d), query_regions (queries*regions x d), region_to_image, query_images)
    as float64 arrays of fp32-rounded unit rows, from one default_rng(seed):
    image centres, region noise, query images, query region noise."""
    rng = np.random.default_rng(cfg.seed)
    centres = rng.standard_normal((cfg.images, cfg.d))
    centres /= np.linalg.norm(centres, axis=1, keepdims=True)
    r2i = np.repeat(np.arange(cfg.images), cfg.regions)
    x = centres[r2i] + cfg.sigma * rng.standard_normal((cfg.n, cfg.d))
    qimg = rng.choice(cfg.images, size=cfg.queries, replace=False)
    qx = centres[np.repeat(qimg, cfg.regions)] + cfg.sigma * rng.standard_normal((cfg.queries * cfg.regions, cfg.d))

    def unit32(a):
        a = a.astype(np.float32).astype(np.float64)
        return a / np.linalg.norm(a, axis=1, keepdims=True)

    return unit32(x), unit32(qx), r2i, qimg


CONFIGS = {
    "C1": Config("C1", 1, 10_000, 128, 100, 0.1, None, 30, 3.0, 300, 50, 3, 0.10, 100, 30),
    "C2": Config("C2", 2, 100_000, 512, 1_000, 0.1, 1.1, 50, 3.0, 2_000, 200, 3, 0.05, 1_000, 50),
    "C3": Config("C3", 3, 1_000_000, 2048, 10_000, 0.1, 1.1, 50, 3.0, 5_000, 500, 3, 0.02, 10_000, 50),
}


def cluster_probabilities(clusters: int, zipf: float | None) -> np.ndarray:
    if zipf is None:
        return np.full(clusters, 1.0 / clusters)
    w = np.arange(1, clusters + 1, dtype=np.float64) ** (-zipf)
    return w / w.sum()


def cluster_descriptors(cfg: Config, n: int | None = None, queries: int | None = None):
    """(data, query_vectors, labels) as float64 arrays of fp32-rounded unit rows.

    Rows are ``normalise(centre[label] + sigma * N(0, I_d))``; the descriptors
    are rounded through float32 ("fp32 descriptors" in BASELINE.json) and then
    renormalised in float64 so they pass the reference's unit-norm check
    (``descriptors.py:41-47``).
    """
    n = cfg.n if n is None else n
    queries = cfg.queries if queries is None else queries
    rng = np.random.default_rng(cfg.seed)
    centres = rng.standard_normal((cfg.clusters, cfg.d))
    centres /= np.linalg.norm(centres, axis=1, keepdims=True)
    p = cluster_probabilities(cfg.clusters, cfg.zipf)
    labels = rng.choice(cfg.clusters, size=n + queries, p=p)
    x = centres[labels] + cfg.sigma * rng.standard_normal((n + queries, cfg.d))
    x = x.astype(np.float32).astype(np.float64)
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    return x[:n], x[n:], labels


def device_cluster_descriptors(cfg: Config, device, n: int | None = None,
                               queries: int | None = None, dtype=None):
    """GPU-side generator with the same model, for configs too big for numpy.

    Returns (data, queries) as unit-norm float32 torch tensors on ``device``.
    Not numpy-identical (there is no CPU oracle at these sizes).
    """
    import torch

    dtype = torch.float32 if dtype is None else dtype
    n = cfg.n if n is None else n
    queries = cfg.queries if queries is None else queries
    g = torch.Generator(device=device)
    g.manual_seed(cfg.seed)
    centres = torch.randn(cfg.clusters, cfg.d, generator=g, device=device)
    centres /= centres.norm(dim=1, keepdim=True)
    p = torch.as_tensor(cluster_probabilities(cfg.clusters, cfg.zipf), device=device)
    total = n + queries
    labels = torch.multinomial(p, total, replacement=True, generator=g)
    out = torch.empty(total, cfg.d, device=device, dtype=dtype)
    step = 1 << 16
    for s in range(0, total, step):
        e = min(total, s + step)
        blk = centres[labels[s:e]] + cfg.sigma * torch.randn(e - s, cfg.d, generator=g, device=device)
        out[s:e] = (blk / blk.norm(dim=1, keepdim=True)).to(dtype)
    return out[:n], out[n:], labels
