"""Seeded synthetic streams for the BASELINE.json configs.

The reference's datagen (proj/src/datagen.cpp) makes sum-of-sines tensors;
the BASELINE configs ask for Tucker-model streams instead, so the generators
here are new. They reuse the reference's exact per-slice noise rule
||N_t||_F = eta * ||X_t||_F (datagen.cpp:78-103).

Every slice t is a deterministic function of (config seed, t): the small
ground-truth pieces (factors, core, time rows) come from numpy PCG64 streams,
so the oracle and the GPU path always see identical bytes. Slices are built
either with numpy (small configs, golden fixtures) or with torch on a CUDA
device (large configs; copied to host when a CPU checker needs them).
Tensors are returned as flat colexicographic (mode-0 fastest) float64 buffers.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

BASE_SEED = 20261019


@dataclass
class StreamConfig:
    name: str
    slice_dims: tuple            # N_0..N_{d-2}
    spatial_ranks: tuple         # ground-truth R_0..R_{d-2}
    time_rank: int
    n_slices: int                # total slices (init + streamed)
    n_init: int
    tau: float
    eta: float
    seed: int
    spectrum_ratio: float = 0.0  # >0: core = G x_k diag(ratio^i) (config 3)
    growth: tuple = ()           # (start, step, every, max): config 5 rank growth
    notes: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def order(self) -> int:
        return len(self.slice_dims) + 1

    @property
    def slice_elems(self) -> int:
        return int(np.prod(self.slice_dims))

    @property
    def slice_bytes(self) -> int:
        return 8 * self.slice_elems


CONFIGS = {
    # configs[0]: CPU-runnable oracle case.
    "c1": StreamConfig("c1", (64, 64), (4, 4), 4, 200, 20, 1e-2, 1e-4, BASE_SEED + 1,
                       notes="3-way, 200 slices of 64x64, ranks (4,4,4)"),
    # configs[1]: the single-GPU headline.
    "c2": StreamConfig("c2", (200, 200, 200), (10, 10, 10), 10, 100, 10, 1e-2, 1e-3,
                       BASE_SEED + 2,
                       notes="4-way, 100 slices of 200^3, spatial ranks 10, R_t=10 (unspecified in BASELINE)"),
    "c3": StreamConfig("c3", (512, 512, 512), (32, 32, 32), 32, 50, 5, 1e-3, 1e-4,
                       BASE_SEED + 3, spectrum_ratio=0.8,
                       notes="4-way, 50 slices of 512^3, core G x_k diag(0.8^i), R_t=32"),
    # configs[3]: combustion-like 5-way stream of advected Gaussian blobs
    # (the HCCI data itself is not in the container; see BlobStream)
    "c4": StreamConfig("c4", (384, 384, 384, 16), (0, 0, 0, 0), 0, 100, 10, 1e-3, 1e-5,
                       BASE_SEED + 4, extra={"kind": "blobs", "n_blobs": 64, "base_res": 384},
                       notes="5-way combustion-like, 100 slices of 384^3 x 16 variables: tanh(a_k f + b_k) "
                             "of 64 advected 3-D Gaussian blobs"),
    "c5": StreamConfig("c5", (256, 256, 256), (36, 36, 36), 36, 400, 10, 1e-4, 1e-6,
                       BASE_SEED + 5, growth=(8, 4, 50, 36),
                       notes="4-way rank growth 8->36 (+4 every 50 slices); nested core, R_t = active rank; init 10 (unspecified)"),
}


def scaled(cfg: StreamConfig, slice_dims: tuple, n_slices: int | None = None,
           n_init: int | None = None, name: str | None = None) -> StreamConfig:
    """Same generator and seeds at a reduced resolution (for CPU parity runs)."""
    ranks = tuple(min(r, n) for r, n in zip(cfg.spatial_ranks, slice_dims))
    return StreamConfig(name or cfg.name + "_small", tuple(slice_dims), ranks, cfg.time_rank,
                        n_slices or cfg.n_slices, n_init or cfg.n_init, cfg.tau, cfg.eta,
                        cfg.seed, cfg.spectrum_ratio,
                        tuple(min(g, min(slice_dims)) for g in cfg.growth) if cfg.growth else (),
                        cfg.notes + " (scaled)", dict(cfg.extra))


def make_stream(cfg: StreamConfig):
    """The generator a config names (Tucker-model streams, or advected blobs)."""
    if cfg.extra.get("kind") == "blobs":
        return BlobStream(cfg)
    return TuckerStream(cfg)


def _rng(seed: int, *stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, *stream])))


class TuckerStream:
    """Ground truth + per-slice synthesis for one config."""

    def __init__(self, cfg: StreamConfig):
        self.cfg = cfg
        R = cfg.spatial_ranks
        self.factors = []
        for k, (n, r) in enumerate(zip(cfg.slice_dims, R)):
            g = _rng(cfg.seed, 1, k).standard_normal((n, r))
            q, rr = np.linalg.qr(g)
            q = q * np.sign(np.diag(rr))[None, :]  # deterministic sign
            self.factors.append(np.ascontiguousarray(q))
        core_dims = tuple(R) + (cfg.time_rank,)
        # core indexed c[i0, i1, ..., it]
        core = _rng(cfg.seed, 2).standard_normal(core_dims)
        if cfg.spectrum_ratio > 0:
            for k in range(len(R)):
                shape = [1] * len(core_dims)
                shape[k] = R[k]
                core = core * (cfg.spectrum_ratio ** np.arange(R[k])).reshape(shape)
        self.core = core

    def active_rank(self, t: int) -> int | None:
        g = self.cfg.growth
        if not g:
            return None
        start, step, every, mx = g
        return min(start + step * (t // every), mx)

    def time_row(self, t: int) -> np.ndarray:
        return _rng(self.cfg.seed, 3, t).standard_normal(self.cfg.time_rank)

    def _slice_core(self, t: int) -> tuple[np.ndarray, list]:
        """Core contracted with the time row. With rank growth (config 5) the
        core is block-nested: time direction j only touches the spatial block
        [:b_j]^(d-1), b_j = the active rank of the epoch that introduced j, and
        slice t only mixes the R(t) directions active at t. Spatial ranks then
        grow 8 -> 36 while the streaming rank stays <= 36."""
        a = self.time_row(t)
        ra = self.active_rank(t)
        core = self.core
        if ra is not None:
            a = a.copy()
            a[ra:] = 0.0
            core = core * self._growth_mask()
        g = np.tensordot(core, a, axes=([core.ndim - 1], [0]))  # R_0 x .. x R_{d-2}
        return g, self.factors

    def _growth_mask(self) -> np.ndarray:
        if getattr(self, "_mask", None) is None:
            start, step, every, mx = self.cfg.growth
            R = self.cfg.spatial_ranks
            mask = np.zeros(tuple(R) + (self.cfg.time_rank,))
            for j in range(self.cfg.time_rank):
                b = start
                while b <= j:
                    b += step
                b = min(b, mx)
                sl = tuple(slice(0, b) for _ in R)
                mask[sl + (j,)] = 1.0
            self._mask = mask
        return self._mask

    def clean_slice_numpy(self, t: int) -> np.ndarray:
        g, facs = self._slice_core(t)
        x = g
        for k, f in enumerate(facs):
            # x_k <- f @ x along mode k
            x = np.moveaxis(np.tensordot(f, x, axes=([1], [k])), 0, k)
        return x

    def noise_numpy(self, t: int) -> np.ndarray:
        return _rng(self.cfg.seed, 4, t).standard_normal(self.cfg.slice_dims)

    def slice_numpy(self, t: int) -> np.ndarray:
        """Slice t as a flat colexicographic float64 buffer."""
        x = self.clean_slice_numpy(t)
        if self.cfg.eta > 0:
            z = self.noise_numpy(t)
            xn, zn = np.linalg.norm(x), np.linalg.norm(z)
            if xn > 0 and zn > 0:
                x = x + (self.cfg.eta * xn / zn) * z
        return np.ascontiguousarray(x.transpose()).ravel()

    def init_numpy(self) -> np.ndarray:
        """Initial batch (d-way, streaming mode last), flat colexicographic."""
        return np.concatenate([self.slice_numpy(t) for t in range(self.cfg.n_init)])

    def init_dims(self) -> list:
        return list(self.cfg.slice_dims) + [self.cfg.n_init]

    # --- torch (device) synthesis for the large configs ---
    def slice_torch(self, t: int, device, generator_seed: int | None = None):
        """Slice t built on `device` with torch (fp64). Noise comes from a torch
        Philox stream seeded by (seed, t): deterministic per device type, but
        not bit-equal to slice_numpy. Returns a flat colexicographic tensor."""
        import torch
        g, facs = self._slice_core(t)
        x = torch.as_tensor(g, dtype=torch.float64, device=device)
        for k, f in enumerate(facs):
            ft = torch.as_tensor(f, dtype=torch.float64, device=device)
            x = torch.movedim(torch.tensordot(ft, x, dims=([1], [k])), 0, k)
        if self.cfg.eta > 0:
            gen = torch.Generator(device=device)
            gen.manual_seed((self.cfg.seed * 1_000_003 + t) & 0x7FFFFFFFFFFFFFFF
                            if generator_seed is None else generator_seed)
            z = torch.randn(x.shape, dtype=torch.float64, device=device, generator=gen)
            x = x + (self.cfg.eta * torch.linalg.vector_norm(x) / torch.linalg.vector_norm(z)) * z
        # colexicographic flat: reverse dims then row-major flatten
        return x.permute(*reversed(range(x.ndim))).contiguous().reshape(-1)


class BlobStream:
    """Config 4 (BASELINE configs[3]): a combustion-like 5-way stream.

    Base field f_t(x, y, z) = sum_b A_b exp(-|p - c_b - v_b t|^2 / (2 w_b^2))
    over 64 seeded 3-D Gaussian blobs: centres uniform in the box, widths
    U[8, 40] cells, velocities N(0, 1) cells/step, amplitudes N(0, 1), no wrap
    (SURVEY §8(d) resolutions of the unspecified distributions). Variable k
    of slice t is tanh(a_k f_t + b_k) with a_k, b_k ~ U(0.5, 2); noise
    ||N_t|| = eta ||X_t|| as for every config. Lengths are in cells of the
    384^3 base grid, so a reduced-resolution `scaled` config draws the same
    field on a coarser grid. Each blob is separable, so f_t is a sum of 64
    outer products (one (N x 64) x (64 x N^2) GEMM on the device).
    """

    def __init__(self, cfg: StreamConfig):
        self.cfg = cfg
        nb = int(cfg.extra.get("n_blobs", 64))
        base = float(cfg.extra.get("base_res", 384))
        dims = cfg.slice_dims[:3]
        self.nvar = cfg.slice_dims[3]
        g = _rng(cfg.seed, 5)
        self.centres = g.uniform(0.0, base, (nb, 3))
        self.widths = g.uniform(8.0, 40.0, nb)
        self.vel = g.standard_normal((nb, 3))
        self.amp = g.standard_normal(nb)
        v = _rng(cfg.seed, 6)
        self.a = v.uniform(0.5, 2.0, self.nvar)
        self.b = v.uniform(0.5, 2.0, self.nvar)
        # grid point i of a dimension with n points sits at (i + 0.5) base / n
        self.coords = [(np.arange(n) + 0.5) * (base / n) for n in dims]

    def profiles(self, t: int) -> list:
        """Per dimension: (n_blobs x N) Gaussian factors of the blobs at time t."""
        out = []
        for d, xs in enumerate(self.coords):
            c = self.centres[:, d] + self.vel[:, d] * t
            out.append(np.exp(-((xs[None, :] - c[:, None]) ** 2) / (2.0 * self.widths[:, None] ** 2)))
        return out

    def clean_slice_numpy(self, t: int) -> np.ndarray:
        gx, gy, gz = self.profiles(t)
        f = np.einsum("b,bx,by,bz->xyz", self.amp, gx, gy, gz, optimize=True)
        return np.stack([np.tanh(self.a[k] * f + self.b[k]) for k in range(self.nvar)], axis=3)

    def noise_numpy(self, t: int) -> np.ndarray:
        return _rng(self.cfg.seed, 4, t).standard_normal(self.cfg.slice_dims)

    slice_numpy = TuckerStream.slice_numpy
    init_numpy = TuckerStream.init_numpy
    init_dims = TuckerStream.init_dims

    def slice_torch(self, t: int, device, generator_seed: int | None = None):
        """Slice t on `device` (fp64), flat colexicographic; same field as
        slice_numpy up to rounding, torch Philox noise (not bit-equal)."""
        import torch
        gx, gy, gz = [torch.as_tensor(p, dtype=torch.float64, device=device) for p in self.profiles(t)]
        nx, ny, nz = gx.shape[1], gy.shape[1], gz.shape[1]
        amp = torch.as_tensor(self.amp, dtype=torch.float64, device=device)
        # colexicographic (x fastest): F[z, y, x] = sum_b (A gz)[b, z] gy[b, y] gx[b, x]
        zy = ((amp[:, None] * gz)[:, :, None] * gy[:, None, :]).reshape(gx.shape[0], nz * ny)
        f = (zy.t() @ gx).reshape(nz, ny, nx)  # (z, y, x) row-major == colexicographic (x, y, z)
        x = torch.empty((self.nvar, nz, ny, nx), dtype=torch.float64, device=device)
        for k in range(self.nvar):
            torch.tanh(f * float(self.a[k]) + float(self.b[k]), out=x[k])
        del f, zy
        if self.cfg.eta > 0:
            gen = torch.Generator(device=device)
            gen.manual_seed((self.cfg.seed * 1_000_003 + t) & 0x7FFFFFFFFFFFFFFF
                            if generator_seed is None else generator_seed)
            xn = torch.linalg.vector_norm(x)
            z = torch.randn(x.shape, dtype=torch.float64, device=device, generator=gen)
            x.add_(z, alpha=float(self.cfg.eta * xn / torch.linalg.vector_norm(z)))
            del z
        return x.reshape(-1)
