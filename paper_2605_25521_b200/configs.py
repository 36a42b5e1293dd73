"""The five BASELINE.json workloads as seeded synthetic generators.

The reference paper measures on SIFT/LAION/SSNPP-style sets that are not
available here; BASELINE.json restates each workload as a seeded
distribution, and these generators implement exactly those descriptions
(SURVEY.md §8(d)).  Rows are generated on the GPU in fixed chunks of
2**20 rows, each chunk from its own Philox stream seeded by
(config seed, chunk index), so any row range -- and therefore any
sharding across 1/2/4/8 GPUs -- sees identical rows.  Mixture centres,
sample indices and Lloyd initial points come from numpy PCG64 streams on
the host.

Definitions fixed here (BASELINE leaves them open):
  * training sample: ``sorted(PCG64(1).choice(N, n_train, replace=False))``
    -- the same rows for every subspace;
  * Lloyd init: the sample's rows at ``sorted(PCG64(2).choice(n_train, 256,
    replace=False))``, cut into subspaces; Lloyd runs with tol = 0;
  * config 1's codebooks: per subspace, 256 distinct data subvectors drawn
    uniformly with PCG64(1) from the sorted unique subvectors.
"""

from __future__ import annotations

from dataclasses import dataclass

import zlib

import numpy as np

CHUNK = 1 << 20


@dataclass(frozen=True)
class PQConfig:
    name: str
    n: int
    d: int
    m: int
    k: int
    dtype: str            # "f32" | "u8"
    dist: str             # "mixture" | "sphere"
    n_comp: int = 0
    lo: float = 0.0
    hi: float = 0.0
    sigma: float = 0.0
    clip_lo: float | None = None
    clip_hi: float | None = None
    rounded: bool = False
    n_train: int = 0
    iters: int = 0
    codebook: str = "lloyd"  # "lloyd" | "sampled"
    batch: int = 0           # streaming batch rows (config 5)
    seed: int = 0

    @property
    def sub(self) -> int:
        return self.d // self.m

    @property
    def elem_bytes(self) -> int:
        return 1 if self.dtype == "u8" else 4

    def flops_per_vec(self) -> int:
        return 2 * self.k * self.d

    def bytes_per_vec(self) -> int:
        return self.d * self.elem_bytes + self.m

    def scaled(self, n: int, n_train: int | None = None) -> "PQConfig":
        from dataclasses import replace
        return replace(self, n=n, n_train=self.n_train if n_train is None else n_train)


CONFIGS = {
    "c1": PQConfig("c1", 100_000, 128, 16, 256, "f32", "mixture", n_comp=64, lo=0, hi=255, sigma=20,
                   clip_lo=0, clip_hi=255, rounded=True, codebook="sampled"),
    "c2": PQConfig("c2", 1_000_000, 960, 120, 256, "f32", "mixture", n_comp=256, lo=0, hi=1, sigma=0.08,
                   clip_lo=0, n_train=100_000, iters=25),
    "c3": PQConfig("c3", 10_000_000, 768, 96, 256, "f32", "sphere", n_train=200_000, iters=10),
    "c4": PQConfig("c4", 200_000_000, 128, 32, 256, "u8", "mixture", n_comp=1024, lo=0, hi=255, sigma=15,
                   clip_lo=0, clip_hi=255, rounded=True, n_train=1_000_000, iters=20),
    "c5": PQConfig("c5", 1_000_000, 1536, 192, 256, "f32", "sphere", n_train=100_000, iters=10, batch=4096),
}


def centres(cfg: PQConfig) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(cfg.seed))
    return rng.uniform(cfg.lo, cfg.hi, size=(cfg.n_comp, cfg.d)).astype(np.float32)


def _chunk_rows(cfg: PQConfig, c: int, rows: int, dev, cen):
    import torch
    g = torch.Generator(device=dev)
    g.manual_seed((cfg.seed * 1_000_003 + zlib.crc32(cfg.name.encode()) * 7919 + c) & 0x7FFFFFFFFFFF)
    if cfg.dist == "sphere":
        x = torch.randn((rows, cfg.d), generator=g, device=dev, dtype=torch.float32)
        x /= torch.linalg.vector_norm(x, dim=1, keepdim=True)
        return x
    lab = torch.randint(0, cfg.n_comp, (rows,), generator=g, device=dev)
    x = torch.randn((rows, cfg.d), generator=g, device=dev, dtype=torch.float32)
    x.mul_(cfg.sigma).add_(cen[lab])
    if cfg.rounded:
        x.round_()
    if cfg.clip_lo is not None or cfg.clip_hi is not None:
        x.clamp_(min=cfg.clip_lo, max=cfg.clip_hi)
    if cfg.dtype == "u8":
        return x.to(torch.uint8)
    return x


def generate(cfg: PQConfig, begin: int, end: int, dev, out=None):
    """Rows [begin, end) of the config's dataset as a CUDA tensor (float32 or
    uint8), generated chunk by chunk on ``dev``."""
    import torch
    dt = torch.uint8 if cfg.dtype == "u8" else torch.float32
    if out is None:
        out = torch.empty((end - begin, cfg.d), dtype=dt, device=dev)
    cen = torch.from_numpy(centres(cfg)).to(dev) if cfg.dist == "mixture" else None
    c0, c1 = begin // CHUNK, (end - 1) // CHUNK if end > begin else begin // CHUNK - 1
    for c in range(c0, c1 + 1):
        lo, hi = c * CHUNK, (c + 1) * CHUNK
        rows = _chunk_rows(cfg, c, CHUNK, dev, cen)
        a, b = max(lo, begin), min(hi, end)
        out[a - begin:b - begin].copy_(rows[a - lo:b - lo])
        del rows
    return out


def sample_indices(cfg: PQConfig) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(1))
    idx = rng.choice(cfg.n, size=cfg.n_train, replace=False)
    idx.sort()
    return idx


def init_indices(cfg: PQConfig) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(2))
    idx = rng.choice(cfg.n_train, size=cfg.k, replace=False)
    idx.sort()
    return idx


def training_sample(cfg: PQConfig, dev):
    """(n_train, d) float32 CUDA tensor: the sampled rows (gathered chunk by
    chunk, so the full dataset never has to be resident)."""
    import torch
    idx = sample_indices(cfg)
    out = torch.empty((cfg.n_train, cfg.d), dtype=torch.float32, device=dev)
    cen = torch.from_numpy(centres(cfg)).to(dev) if cfg.dist == "mixture" else None
    chunk_of = idx // CHUNK
    pos = 0
    for c in np.unique(chunk_of):
        sel = idx[chunk_of == c] - c * CHUNK
        rows = _chunk_rows(cfg, int(c), CHUNK, dev, cen)
        out[pos:pos + sel.shape[0]] = rows[torch.from_numpy(sel).to(dev)].float()
        pos += sel.shape[0]
        del rows
    return out


def subspace_major(X, m: int):
    """(n, d) -> (m, n, d/m) contiguous: the layout of the Lloyd kernels."""
    n, d = X.shape
    return X.reshape(n, m, d // m).permute(1, 0, 2).contiguous()


def lloyd_init(cfg: PQConfig, sample_sm) -> np.ndarray:
    """(m, k, sub) float64 initial centroids: the init rows of the sample."""
    import torch
    ii = torch.from_numpy(init_indices(cfg)).to(sample_sm.device)
    return sample_sm[:, ii, :].double().cpu().numpy()


def sampled_codebooks(cfg: PQConfig, X_host: np.ndarray) -> np.ndarray:
    """Config 1: per subspace 256 distinct data subvectors, drawn with PCG64(1)."""
    rng = np.random.Generator(np.random.PCG64(1))
    sub = cfg.sub
    out = np.empty((cfg.m, cfg.k, sub), np.float32)
    for j in range(cfg.m):
        u = np.unique(X_host[:, j * sub:(j + 1) * sub], axis=0)
        out[j] = u[np.sort(rng.choice(u.shape[0], cfg.k, replace=False))]
    return out
