"""Seeded synthetic matrix streams for the BASELINE.json configs (C1..C5).

This module holds NO arithmetic of the method (no Gram, no eigensolver, no
SCW).  It only draws the input streams A_d (m x n, fp32) that both the float64
oracle (``oracle/``) and the CUDA path consume.  The paper's datasets (HSI,
Logo, MRI; Table 1) are not available, so these streams
stand in for them ("Input recipe").

Recipe (BASELINE.json ``configs``; SURVEY.md §8(d) "Proposed generator"):

* shared factor: U0 = Q of QR(N(0,1)^{m x p}) with sign(diag R) > 0,
* per matrix d (global stream index g = d for training, D_train + d for test):
  K_g = (N - N^T)/2 with N ~ N(0,1)^{m x m}   (random skew matrix),
  U_g = exp(h K_g) U0, evaluated as a truncated Taylor action (TAYLOR_TERMS),
  V_g = Q of QR(N(0,1)^{n x p}), independent per g,
  A_g = U_g diag(sigma) V_g^T + eta N(0,1)^{m x n},
  frame-like configs (C3, C4): A_g = clip(offset + ..., 0, 1).
* Train/test split in stream order ("past data ... training
  set, future input matrices ... test set"): the first D_train matrices train, the next
  D_test test.

Every matrix is drawn from its own torch.Generator seeded from (seed, g), so any
d-range (a rank's shard, a sampled subset) can be generated independently.  The
draws are made on ``device``; bytes differ between a CPU and a CUDA draw, so a
test always hands the SAME generated array to both sides (copying it across).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import torch

TAYLOR_TERMS = 24
ROTATION_H = 0.05


@dataclasses.dataclass(frozen=True)
class StreamConfig:
    name: str
    m: int
    n: int
    D_train: int
    D_test: int
    k: int
    r: int
    p: int                    # rank of the drifting subspace
    sigma_kind: str           # "geom": sigma_i = s0 * q**i ; "planted": see _sigma
    s0: float
    q: float
    eta: float                # noise level
    offset: Optional[float]   # frame-like: offset then clip to [0, 1]
    drift: bool = True        # U_d = exp(hK_d) U0 (True) or U_d = U0 (False)
    identical: bool = False   # every A_d equals A_0 (PAPER.md:147 special case)
    gap: float = 0.0          # planted eigengap lambda_k/lambda_{k+1} target ("planted")

    def replace(self, **kw) -> "StreamConfig":
        return dataclasses.replace(self, **kw)

    @property
    def train_bytes(self) -> int:
        return 4 * self.m * self.n * self.D_train


def _frame_s0(m: int, n: int, p: int, q: float) -> float:
    # sum_i sigma_i^2 = 0.0144 m n  (RMS 0.12 signal around the 0.5 offset)
    s = sum(q ** (2 * i) for i in range(p))
    return math.sqrt(0.0144 * m * n / s)


CONFIGS = {
    # BASELINE.json configs[0]
    "C1": StreamConfig("C1", 64, 48, 20, 10, 10, 5, 8, "geom", 10.0, 0.7, 0.01, None),
    # configs[1]
    "C2": StreamConfig("C2", 256, 256, 200, 100, 20, 10, 32, "geom", 1.0, 0.9, 0.05, None),
    # configs[2]: rank-64 = 63 drifting directions + the 0.5 mean
    "C3": StreamConfig("C3", 1024, 768, 400, 200, 40, 20, 63, "geom",
                       _frame_s0(1024, 768, 63, 0.95), 0.95, 0.02, 0.5),
    # configs[3]: rank-96 = 95 drifting directions + the mean
    "C4": StreamConfig("C4", 1080, 1920, 2000, 500, 60, 30, 95, "geom",
                       _frame_s0(1080, 1920, 95, 0.95), 0.95, 0.02, 0.5),
    # configs[4]
    "C5": StreamConfig("C5", 4096, 4096, 2000, 256, 100, 50, 256, "geom", 1.0, 0.98, 0.01, None),
}


def planted(base: str | StreamConfig, gap: float = 1.2, D_train: Optional[int] = None,
            D_test: Optional[int] = None) -> StreamConfig:
    """Gap-planted variant: no drift, small noise, sigma chosen so the
    training Gram has lambda_k / lambda_{k+1} ~= gap, which makes the projector parity
    check bind (BASELINE.json: projector tolerance applies when the gap >= 1.05)."""
    c = CONFIGS[base] if isinstance(base, str) else base
    p = min(c.k + 8, c.m, c.n)
    return c.replace(name=c.name + f"-planted{gap:g}", p=p, sigma_kind="planted", s0=1.0,
                     q=0.97, eta=1e-3, offset=None, drift=False, gap=gap,
                     D_train=D_train or c.D_train, D_test=D_test or c.D_test)


def identical(base: str | StreamConfig, D_train: Optional[int] = None) -> StreamConfig:
    """All training slices equal: span S must equal span U_k(A)."""
    c = CONFIGS[base] if isinstance(base, str) else base
    return c.replace(name=c.name + "-identical", identical=True, D_train=D_train or c.D_train)


def lowrank(base: str | StreamConfig, rank: Optional[int] = None) -> StreamConfig:
    """Exactly low rank, noise-free, no drift: A_d = U0 diag(sigma) V_d^T with rank p <= r.
    SCW with the trained S must return A exactly (error 0; PAPER.md:149-153 with eps = 0)."""
    c = CONFIGS[base] if isinstance(base, str) else base
    p = rank if rank is not None else min(c.r, 8)
    return c.replace(name=c.name + f"-lowrank{p}", p=p, eta=0.0, offset=None, drift=False)


def _sigma(c: StreamConfig) -> torch.Tensor:
    i = torch.arange(c.p, dtype=torch.float64)
    if c.sigma_kind == "geom":
        return c.s0 * c.q ** i
    # planted: lambda_i ~ D sigma_i^2 for i < p; put a factor `gap` between i = k-1 and k
    s = c.q ** i
    s[c.k:] = s[c.k:] / math.sqrt(c.gap)
    return s


def _gen(seed: int, stream_index: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    # distinct, reproducible 63-bit seeds per (seed, stream index); index -1 = shared draws
    g.manual_seed((seed * 0x9E3779B1 + (stream_index + 1) * 0x85EBCA77) % (2 ** 63 - 1))
    return g


def _orthonormal(rows: int, cols: int, g: torch.Generator, device) -> torch.Tensor:
    x = torch.randn(rows, cols, generator=g, device=device, dtype=torch.float64)
    q, r = torch.linalg.qr(x)
    sgn = torch.sign(torch.diagonal(r))
    sgn[sgn == 0] = 1.0
    return q * sgn


def shared_basis(c: StreamConfig, seed: int = 0, device="cpu") -> torch.Tensor:
    """U0 (m x p), the shared subspace every stream matrix rotates."""
    return _orthonormal(c.m, c.p, _gen(seed, -1, device), device)


def _one(c: StreamConfig, seed: int, g_index: int, U0: torch.Tensor, sigma: torch.Tensor,
         device) -> torch.Tensor:
    g = _gen(seed, g_index, device)
    if c.drift:
        K = torch.randn(c.m, c.m, generator=g, device=device, dtype=torch.float64)
        K = 0.5 * (K - K.T)
        hK = ROTATION_H * K
        U = U0.clone()
        T = U0
        for j in range(1, TAYLOR_TERMS + 1):
            T = (hK @ T) / j
            U = U + T
    else:
        U = U0
    V = _orthonormal(c.n, c.p, g, device)
    A = (U * sigma) @ V.T
    if c.eta != 0.0:
        A = A + c.eta * torch.randn(c.m, c.n, generator=g, device=device, dtype=torch.float64)
    if c.offset is not None:
        A = torch.clamp(A + c.offset, 0.0, 1.0)
    return A.to(torch.float32)


def generate(c: StreamConfig | str, split: str = "train", start: int = 0, stop: Optional[int] = None,
             seed: int = 0, device="cpu", out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Matrices [start, stop) of the training (split="train") or test stream as one
    contiguous fp32 tensor [stop-start, m, n] (slice-major, row-major within a slice)."""
    if isinstance(c, str):
        c = CONFIGS[c]
    total = c.D_train if split == "train" else c.D_test
    stop = total if stop is None else stop
    if not (0 <= start <= stop <= total):
        raise ValueError(f"range [{start},{stop}) outside {split} stream of {total}")
    base = 0 if split == "train" else c.D_train
    U0 = shared_basis(c, seed, device)
    sigma = _sigma(c).to(device)
    if out is None:
        out = torch.empty(stop - start, c.m, c.n, dtype=torch.float32, device=device)
    if c.identical:
        a0 = _one(c, seed, 0, U0, sigma, device)
        out.copy_(a0.expand(stop - start, c.m, c.n))
        return out
    for i, d in enumerate(range(start, stop)):
        out[i].copy_(_one(c, seed, base + d, U0, sigma, device))
    return out



# ------------------------------------------------------------------ random-sketch baselines (f3)
# Draws only (no method arithmetic): the untrained sketches the paper compares against in spirit
# ("generated randomly from some distribution, such as Gaussian"; IVY's "sparse random
# sign matrix" initialisation).  Both feed the SAME SCW kernels as the trained
# S: Algorithm 1 only uses rowspace(S A), so S need not have orthonormal rows.

def random_sign_sketch(k: int, m: int, seed: int = 0) -> torch.Tensor:
    """[k][m] fp32 CountSketch pattern: every column has exactly one nonzero, +-1, in a uniformly
    random row (the sparsity level is a decision, not the paper's)."""
    if not (1 <= k <= m):
        raise ValueError("need 1 <= k <= m")
    g = torch.Generator().manual_seed(int(seed) * 1_000_003 + 17)
    rows = torch.randint(0, k, (m,), generator=g)
    signs = torch.randint(0, 2, (m,), generator=g).to(torch.float32) * 2.0 - 1.0
    S = torch.zeros(k, m, dtype=torch.float32)
    S[rows, torch.arange(m)] = signs
    return S


def random_gaussian_sketch(k: int, m: int, seed: int = 0) -> torch.Tensor:
    """[k][m] fp32 with i.i.d. N(0, 1/k) entries."""
    if not (1 <= k <= m):
        raise ValueError("need 1 <= k <= m")
    g = torch.Generator().manual_seed(int(seed) * 1_000_003 + 29)
    return (torch.randn(k, m, generator=g, dtype=torch.float64) / math.sqrt(k)).to(torch.float32)


# Start block of the matrix-free (randomized block Krylov) sketch: the random
# numbers that method draws, passed in as an input so the GPU path and the oracle start alike.

def start_block(m: int, p: int, seed: int = 0) -> torch.Tensor:
    """[m][p] fp64 with i.i.d. N(0, 1) entries."""
    if m < 1 or p < 1:
        raise ValueError("need m, p >= 1")
    g = torch.Generator().manual_seed(int(seed) * 1_000_003 + 41)
    return torch.randn(m, p, generator=g, dtype=torch.float64)
