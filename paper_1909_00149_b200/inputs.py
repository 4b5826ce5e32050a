"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NO arithmetic of the method (no divergence, shrinkage, step
or dual update): it only draws frames.  It is the one module both sides may
use; ``oracle/`` never imports it, the tests pass
its arrays to both sides.

The five configurations are BASELINE.json ``configs[0..4]`` (C1..C5).  Where
BASELINE.json leaves a generator detail open, the choice is DESIGN.md reading
L20 ("proposed").  Every draw uses numpy PCG64 seeded with
``SeedSequence([config_seed, item...])`` so any frame or pair can be produced
alone, on any rank, bit-identically.  Values are produced in float64 and
returned as float32 (the precision the kernels consume).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    n_chains: int          # B
    n_frames: int          # T (pairs P = T-1 per chain)
    ny: int
    nx: int
    iters: int
    alpha: float
    seed: int
    rho: float = math.inf  # fixed marginals unless stated
    note: str = ""

    @property
    def n_pairs(self) -> int:
        return self.n_chains * (self.n_frames - 1)

    @property
    def px_iters(self) -> int:
        return self.n_pairs * self.nx * self.ny * self.iters


CONFIGS = {
    "C1": Config("C1", 1, 2, 64, 64, 500, 0.5, 0, note="BASELINE configs[0]: blob shifted (3,2) px, x1.1"),
    "C2": Config("C2", 1, 2, 512, 512, 2000, 0.3, 2, note="BASELINE configs[1]: 16 blobs + 1% sparse noise"),
    "C3": Config("C3", 1, 64, 256, 256, 1000, 2.0, 3, note="BASELINE configs[2]: T=64 video, alpha=2 (L15)"),
    "C4": Config("C4", 1, 256, 1024, 1024, 500, 2.0, 4, note="BASELINE configs[3]: T=256 video, alpha=2 (L15)"),
    "C5": Config("C5", 64, 2, 4096, 4096, 300, 0.2, 5, note="BASELINE configs[4]: 64 independent warped pairs"),
}


def _rng(*items) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(v) for v in items])))


def _gauss2(ny, nx, cy, cx, sy, sx=None, theta=0.0):
    """Elliptical Gaussian profile exp(-d^2/2) with 1-sigma semi-axes (sx, sy)
    rotated by theta, evaluated at pixel centres (j, i)."""
    sx = sy if sx is None else sx
    j = np.arange(ny, dtype=np.float64)[:, None] - cy
    i = np.arange(nx, dtype=np.float64)[None, :] - cx
    c, s = math.cos(theta), math.sin(theta)
    u = c * i + s * j
    v = -s * i + c * j
    return np.exp(-0.5 * ((u / sx) ** 2 + (v / sy) ** 2))


def _stamp(img, cy, cx, sa, sb, theta, amp, reach=4.0):
    """Add amp * elliptical Gaussian to img, evaluated on its +-reach*sigma box."""
    ny, nx = img.shape
    R = reach * max(sa, sb)
    j0, j1 = max(0, int(math.floor(cy - R))), min(ny, int(math.ceil(cy + R)) + 1)
    i0, i1 = max(0, int(math.floor(cx - R))), min(nx, int(math.ceil(cx + R)) + 1)
    if j0 >= j1 or i0 >= i1:
        return
    img[j0:j1, i0:i1] += amp * _gauss2(j1 - j0, i1 - i0, cy - j0, cx - i0, sb, sa, theta)


def _reflect(v, n):
    """Reflect a coordinate into [0, n-1] (blobs bounce off the frame edge)."""
    L = float(n - 1)
    v = math.fmod(abs(v), 2 * L)
    return 2 * L - v if v > L else v


# ------------------------------------------------------------------------------- C1
def gen_c1() -> np.ndarray:
    """configs[0]: x0 = Gaussian blob sigma 4 px, peak 1 at (32,32) (proposed
    centre); x1 = 1.1 * same blob shifted by (dx=+3 along i, dy=+2 along j) (L5)."""
    x0 = _gauss2(64, 64, 32.0, 32.0, 4.0)
    x1 = 1.1 * _gauss2(64, 64, 34.0, 35.0, 4.0)
    return np.stack([x0, x1])[None].astype(np.float32)


# ------------------------------------------------------------------------------- C2
def gen_c2(seed: int = 2, n: int = 512, n_blobs: int = 16) -> np.ndarray:
    """configs[1]: 16 blobs, centres U[0,n)^2, sigma U[3,12], amplitude U[0.2,1];
    x1 moves each blob by radius U[0,8] at angle U[0,2pi) (sub-pixel, analytic)
    and scales it by U[0.8,1.25]; '1% sparse uniform noise' = independent
    Bernoulli(0.01) mask per frame adding U[0,1) (L20)."""
    g = _rng(seed, 0)
    cy, cx = g.uniform(0, n, n_blobs), g.uniform(0, n, n_blobs)
    sig = g.uniform(3, 12, n_blobs)
    amp = g.uniform(0.2, 1.0, n_blobs)
    rad, ang = g.uniform(0, 8, n_blobs), g.uniform(0, 2 * math.pi, n_blobs)
    gain = g.uniform(0.8, 1.25, n_blobs)
    frames = np.zeros((2, n, n))
    for b in range(n_blobs):
        _stamp(frames[0], cy[b], cx[b], sig[b], sig[b], 0.0, amp[b])
        _stamp(frames[1], cy[b] + rad[b] * math.sin(ang[b]), cx[b] + rad[b] * math.cos(ang[b]),
               sig[b], sig[b], 0.0, amp[b] * gain[b])
    for t in range(2):
        h = _rng(seed, 1, t)
        mask = h.random((n, n)) < 0.01
        frames[t] += mask * h.random((n, n))
    return frames[None].astype(np.float32)


# ------------------------------------------------------------------------------- C3
def gen_c3(seed: int = 3, n: int = 256, T: int = 64, n_blobs: int = 8) -> np.ndarray:
    """configs[2]: 8 blobs (sigma U[3,8]) on linear trajectories, speed U[1,3]
    px/frame, angle U[0,2pi), centres U[32,224]^2 (bouncing off edges);
    intensity A_b (1 + 0.2 sin(2 pi t / P_b + phi_b)), A_b U[0.5,1], P_b U[16,64];
    static background U V^T / (2R), R = 2, U, V entries U[0,1], values in
    [0, 0.5] (the UV^T/4R protocol of P:930 rescaled to the stated range) (L20)."""
    g = _rng(seed, 0)
    cy, cx = g.uniform(32, 224, n_blobs) * n / 256, g.uniform(32, 224, n_blobs) * n / 256
    sig = g.uniform(3, 8, n_blobs)
    spd, ang = g.uniform(1, 3, n_blobs), g.uniform(0, 2 * math.pi, n_blobs)
    A, Pb, ph = g.uniform(0.5, 1, n_blobs), g.uniform(16, 64, n_blobs), g.uniform(0, 2 * math.pi, n_blobs)
    R = 2
    U, V = g.uniform(0, 1, (n, R)), g.uniform(0, 1, (n, R))
    bg = (U @ V.T) / (2 * R)
    frames = np.empty((T, n, n))
    for t in range(T):
        img = bg.copy()
        for b in range(n_blobs):
            y = _reflect(cy[b] + t * spd[b] * math.sin(ang[b]), n)
            x = _reflect(cx[b] + t * spd[b] * math.cos(ang[b]), n)
            _stamp(img, y, x, sig[b], sig[b], 0.0, A[b] * (1 + 0.2 * math.sin(2 * math.pi * t / Pb[b] + ph[b])))
        frames[t] = img
    return frames[None].astype(np.float32)


# ------------------------------------------------------------------------------- C4
@dataclass
class C4Blobs:
    cy: np.ndarray
    cx: np.ndarray
    sa: np.ndarray
    sb: np.ndarray
    th0: np.ndarray
    om: np.ndarray
    vy: np.ndarray
    vx: np.ndarray
    amp: np.ndarray = field(repr=False)   # [T][n_blobs] intensity random walk


def _c4_blobs(seed: int, n: int, T: int, n_blobs: int) -> C4Blobs:
    g = _rng(seed, 0)
    cy, cx = g.uniform(0, n, n_blobs), g.uniform(0, n, n_blobs)
    sa = g.uniform(5, 30, n_blobs)
    sb = np.array([g.uniform(5, a) for a in sa])
    th0, om = g.uniform(0, math.pi, n_blobs), g.uniform(-0.05, 0.05, n_blobs)
    spd, ang = g.uniform(0, 4, n_blobs), g.uniform(0, 2 * math.pi, n_blobs)
    amp = np.empty((T, n_blobs))
    amp[0] = g.uniform(0.5, 1.0, n_blobs)
    for t in range(1, T):
        amp[t] = np.clip(amp[t - 1] * (1 + g.uniform(-0.02, 0.02, n_blobs)), 0.2, 1.5)
    return C4Blobs(cy, cx, sa, sb, th0, om, spd * np.sin(ang), spd * np.cos(ang), amp)


def gen_c4_frames(t0: int, t1: int, seed: int = 4, n: int = 1024, T: int = 256,
                  n_blobs: int = 32) -> np.ndarray:
    """configs[3] frames t0..t1-1: 32 rotating elliptical blobs, 1-sigma
    semi-axes a U[5,30], b U[5,a], angle theta0 U[0,pi) + omega t, omega
    U[-0.05,0.05] rad/frame, translation speed U[0,4] px/frame (bouncing),
    intensity random walk A_{t+1} = A_t (1 + U[-0.02,0.02]) clipped to
    [0.2, 1.5]; additive iid N(0, 0.02^2) noise, not clipped (L20).
    Returns [1][t1-t0][n][n] float32; frame t depends only on (seed, t)."""
    bl = _c4_blobs(seed, n, T, n_blobs)
    out = np.empty((t1 - t0, n, n), dtype=np.float32)
    for k, t in enumerate(range(t0, t1)):
        img = np.zeros((n, n))
        for b in range(n_blobs):
            y = _reflect(bl.cy[b] + t * bl.vy[b], n)
            x = _reflect(bl.cx[b] + t * bl.vx[b], n)
            _stamp(img, y, x, bl.sa[b], bl.sb[b], bl.th0[b] + bl.om[b] * t, bl.amp[t, b])
        img += _rng(seed, 1, t).normal(0.0, 0.02, (n, n))
        out[k] = img
    return out[None]


def gen_c4(seed: int = 4, n: int = 1024, T: int = 256) -> np.ndarray:
    return gen_c4_frames(0, T, seed=seed, n=n, T=T)


# ------------------------------------------------------------------------------- C5
def _lowpass_field(g: np.random.Generator, n: int, kmax: int) -> np.ndarray:
    """Uniform noise low-pass filtered to modes max(|kx|,|ky|) <= kmax.

    The Fourier coefficients of iid U[0,1) noise are (by the CLT) iid complex
    Gaussian away from DC, so the band-limited field is synthesised directly
    from random coefficients in the kept band (separable inverse DFT) instead
    of filtering n^2 samples -- same distribution, O(n^2 kmax) work (L20)."""
    ks = np.arange(-kmax, kmax + 1)
    C = g.normal(size=(ks.size, ks.size)) + 1j * g.normal(size=(ks.size, ks.size))
    pos = np.arange(n) / n
    Ey = np.exp(2j * math.pi * np.outer(pos, ks))   # [n][K]
    Ex = np.exp(2j * math.pi * np.outer(ks, pos))   # [K][n]
    return np.real(Ey @ C @ Ex)


def _rescale(v, lo, hi):
    mn, mx = v.min(), v.max()
    return lo + (hi - lo) * (v - mn) / (mx - mn)


def gen_c5_pair(b: int, seed: int = 5, n: int = 4096) -> np.ndarray:
    """configs[4] pair b: x0 = low-passed uniform noise (cutoff n/64 cycles per
    grid, 'cutoff 1/64 of grid'), rescaled to [0,1]; displacement D = two
    independent fields under the same filter scaled so max ||D|| = 6 px;
    x1(p) = G(p) x0(p - D(p)) with bilinear sampling and clamped edges; gain G
    under the same filter mapped to [0.7, 1.3] (L20).  Returns [2][n][n] f32."""
    g = _rng(seed, b)
    kmax = max(1, n // 64)
    x0 = _rescale(_lowpass_field(g, n, kmax), 0.0, 1.0)
    dy, dx = _lowpass_field(g, n, kmax), _lowpass_field(g, n, kmax)
    s = 6.0 / np.sqrt(dy * dy + dx * dx).max()
    dy, dx = dy * s, dx * s
    G = _rescale(_lowpass_field(g, n, kmax), 0.7, 1.3)
    jj, ii = np.meshgrid(np.arange(n, dtype=np.float64), np.arange(n, dtype=np.float64), indexing="ij")
    sy = np.clip(jj - dy, 0, n - 1)
    sx = np.clip(ii - dx, 0, n - 1)
    j0 = np.minimum(np.floor(sy).astype(np.int64), n - 2)
    i0 = np.minimum(np.floor(sx).astype(np.int64), n - 2)
    wy, wx = sy - j0, sx - i0
    v = ((1 - wy) * (1 - wx) * x0[j0, i0] + (1 - wy) * wx * x0[j0, i0 + 1]
         + wy * (1 - wx) * x0[j0 + 1, i0] + wy * wx * x0[j0 + 1, i0 + 1])
    x1 = G * v
    return np.stack([x0, x1]).astype(np.float32)


def gen_c5(pairs=range(8), seed: int = 5, n: int = 4096) -> np.ndarray:
    """[len(pairs)][2][n][n]: the pairs of configs[4] with the given indices."""
    return np.stack([gen_c5_pair(b, seed, n) for b in pairs])


# ------------------------------------------------------------------------------- small cases
def gen_random(B: int, T: int, ny: int, nx: int, seed: int, kind: str = "uniform") -> np.ndarray:
    """Generic seeded test frames [B][T][ny][nx] (tiny parity / edge cases).
    kind: 'uniform' U[0,1); 'sparse' 10% of pixels U[0,1) else 0; 'signed' N(0,1)."""
    g = _rng(seed, B, T, ny, nx)
    if kind == "uniform":
        v = g.random((B, T, ny, nx))
    elif kind == "sparse":
        v = g.random((B, T, ny, nx)) * (g.random((B, T, ny, nx)) < 0.1)
    elif kind == "signed":
        v = g.normal(size=(B, T, ny, nx))
    else:
        raise ValueError(kind)
    return v.astype(np.float32)


def gen_two_delta(ny: int, nx: int, p_at, q_at, m_p: float = 1.0, m_q: float = 1.0) -> np.ndarray:
    """Unit (or m_p / m_q) deltas at pixel p_at=(j,i) in x0 and q_at in x1."""
    f = np.zeros((1, 2, ny, nx), dtype=np.float32)
    f[0, 0][p_at] = m_p
    f[0, 1][q_at] = m_q
    return f


# ------------------------------------------------------------------------------- Algorithm 3 (RPCA)
def gen_rpca(T: int, ny: int, nx: int, seed: int, K: int = 5, R: int = 1, noise: float = 0.001,
             observed: float = 0.6, mass_rate: float = 1.0):
    """Synthetic RPCA+UOT-DF instance after the paper's protocol with a
    DIAGONAL Phi stand-in (dense Gaussian Phi is out of scope):
    K targets of intensity U[0.5,1.5] in s_1, each moving by a random step in
    {-1,0,1}^2 per frame (bouncing) with intensity drift U[-mass_rate,mass_rate]*0.1 per
    frame clipped to [0.5,1.5]; L = U V^T/(4R), U, V entries U(0,1); Phi_t =
    diag(m_t) with m_t a Bernoulli(observed) mask (observed = the compression ratio M/N,
    P:957); y_t = Phi_t(s_t + l_t) + N(0, noise^2).  Returns (Y, phi, S, L) float32
    [T][ny][nx]."""
    g = _rng(seed, 77, T, ny, nx)
    S = np.zeros((T, ny, nx))
    pos = np.stack([g.integers(0, ny, K), g.integers(0, nx, K)], axis=1)
    amp = g.uniform(0.5, 1.5, K)
    for t in range(T):
        for k in range(K):
            S[t, pos[k, 0], pos[k, 1]] += amp[k]
        pos = pos + g.integers(-1, 2, (K, 2))
        pos[:, 0] = np.abs(pos[:, 0]) % (2 * ny)
        pos[:, 0] = np.where(pos[:, 0] >= ny, 2 * ny - 1 - pos[:, 0], pos[:, 0])
        pos[:, 1] = np.abs(pos[:, 1]) % (2 * nx)
        pos[:, 1] = np.where(pos[:, 1] >= nx, 2 * nx - 1 - pos[:, 1], pos[:, 1])
        amp = np.clip(amp + 0.1 * mass_rate * g.uniform(-1, 1, K), 0.5, 1.5)
    U, V = g.uniform(0, 1, (ny * nx, R)), g.uniform(0, 1, (T, R))
    L = ((U @ V.T) / (4 * R)).T.reshape(T, ny, nx)
    phi = (g.random((T, ny, nx)) < observed).astype(np.float64)
    Y = phi * (S + L) + noise * g.normal(size=(T, ny, nx))
    f = lambda a: a.astype(np.float32)
    return f(Y), f(phi), f(S), f(L)


def generate(name: str, **kw) -> np.ndarray:
    """Frames [B][T][ny][nx] float32 of config `name` (C5: 8 pairs by default)."""
    if name == "C1":
        return gen_c1()
    if name == "C2":
        return gen_c2(**kw)
    if name == "C3":
        return gen_c3(**kw)
    if name == "C4":
        return gen_c4(**kw)
    if name == "C5":
        return gen_c5(**kw)
    raise KeyError(name)
