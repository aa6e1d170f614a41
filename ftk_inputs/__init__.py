"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the tracking method (no quantisation, gradient, SoS, mesh or
union-find): it only produces scalar fields and their analytic ground truth.  Both sides of every
parity test read the same bytes produced here.

Fields:

* woven 2D:  f = cos(x cos t - y sin t) * sin(x sin t + y cos t)
  x = (i/(nx-1) - 1/2) L, y = (j/(ny-1) - 1/2) L, t = k dt, dt = (h/2) / (L/sqrt 2), h = L/(nx-1).
  Paper density: h = 15/127 (the paper's 128^2 grid over [-7.5, 7.5]^2) at every size.
  Optional Gaussian noise sigma from a counter-based generator (splitmix64 of the
  global linear vertex id, Box-Muller), seed 0.
* moving extremum: f = sum_a sign_a (x_a - c_a(t))^2 on integer grid
  coordinates, c(t) = c0 + v t with dyadic v, so f * 2^8 is an integer and fp32 holds it exactly.
* woven 3D (our choice, not in the paper): f = cos X sin Y + cos z with (X, Y) the rotated woven
  coordinates and z = (k/(nz-1) - 1/2) L.

Every generator computes in float64 (torch, on any device) and casts to the requested dtype.
Layout: [t][y][x] (2D) or [t][z][y][x] (3D), x fastest.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field as dc_field

import torch

PAPER_H = 15.0 / 127.0

_M64 = (1 << 64) - 1


def _i64(v: int) -> int:
    v &= _M64
    return v - (1 << 64) if v >= (1 << 63) else v


def _srl(x: torch.Tensor, k: int) -> torch.Tensor:
    """logical right shift of int64 tensors"""
    return (x >> k) & ((1 << (64 - k)) - 1)


def splitmix64(x: torch.Tensor) -> torch.Tensor:
    """splitmix64 finaliser on int64 tensors (two's-complement wrap-around)."""
    x = x + _i64(0x9E3779B97F4A7C15)
    x = (x ^ _srl(x, 30)) * _i64(0xBF58476D1CE4E5B9)
    x = (x ^ _srl(x, 27)) * _i64(0x94D049BB133111EB)
    return x ^ _srl(x, 31)


def splitmix64_ref(x: int) -> int:
    """pure-Python reference of splitmix64 (for the generator's own unit test)"""
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def gaussian_noise(lin_id: torch.Tensor, seed: int) -> torch.Tensor:
    """N(0,1) per global linear vertex id (int64 tensor): splitmix64 -> two 32-bit uniforms ->
    Box-Muller."""
    z = splitmix64(lin_id + _i64(seed * 0x632BE59BD9B4E019))
    hi = _srl(z, 32).to(torch.float64)
    lo = (z & 0xFFFFFFFF).to(torch.float64)
    u1 = (hi + 0.5) / 4294967296.0
    u2 = (lo + 0.5) / 4294967296.0
    return torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(2.0 * math.pi * u2)


@dataclass
class Woven:
    nx: int
    ny: int
    nt: int
    L: float | None = None       # domain width; None = paper density h = 15/127
    sigma: float = 0.0
    seed: int = 0
    nz: int = 1                  # > 1 selects the 3D woven variant
    scale_log2: int = 26

    @property
    def h(self) -> float:
        return PAPER_H if self.L is None else self.L / (self.nx - 1)

    @property
    def width(self) -> float:
        return self.h * (self.nx - 1) if self.L is None else self.L

    @property
    def dt(self) -> float:
        return 0.5 * self.h / (self.width / math.sqrt(2.0))

    def coords(self, device):
        L = self.width
        xs = (torch.arange(self.nx, dtype=torch.float64, device=device) / (self.nx - 1) - 0.5) * L
        ys = (torch.arange(self.ny, dtype=torch.float64, device=device) / (self.ny - 1) - 0.5) * L
        return xs, ys

    def plane(self, t_global: int, device="cpu") -> torch.Tensor:
        """float64 plane [ny, nx] (2D) or [nz, ny, nx] (3D) at global timestep t_global"""
        xs, ys = self.coords(device)
        t = t_global * self.dt
        c, s = math.cos(t), math.sin(t)
        Y, X = torch.meshgrid(ys, xs, indexing="ij")
        f = torch.cos(X * c - Y * s) * torch.sin(X * s + Y * c)
        if self.nz > 1:
            zs = (torch.arange(self.nz, dtype=torch.float64, device=device) / (self.nz - 1) - 0.5) * self.width
            f = f[None, :, :] + torch.cos(zs)[:, None, None]
        if self.sigma:
            nplane = self.nx * self.ny * self.nz
            lin = torch.arange(nplane, dtype=torch.int64, device=device) + t_global * nplane
            f = f + self.sigma * gaussian_noise(lin, self.seed).reshape(f.shape)
        return f

    def generate(self, t0: int = 0, nt: int | None = None, device="cpu", dtype=torch.float32,
                 out: torch.Tensor | None = None) -> torch.Tensor:
        nt = self.nt - t0 if nt is None else nt
        shape = (nt, self.ny, self.nx) if self.nz == 1 else (nt, self.nz, self.ny, self.nx)
        if out is None:
            out = torch.empty(shape, dtype=dtype, device=device)
        for k in range(nt):
            out[k] = self.plane(t0 + k, device).to(dtype)
        return out

    def analytic_cps_t0(self):
        """Analytic critical points of cos x sin y at t = 0 inside the open domain (2D):
        extrema at (k pi, pi/2 + m pi) (f = +-1), saddles at (pi/2 + k pi, m pi).
        Returns list of (x_grid, y_grid, kind) with kind in {'max','min','saddle'}."""
        L = self.width
        half = L / 2
        out = []
        kmax = int(half / (math.pi / 2)) + 2
        for i in range(-2 * kmax, 2 * kmax + 1):
            for j in range(-2 * kmax, 2 * kmax + 1):
                X = i * math.pi / 2
                Y = j * math.pi / 2
                if not (-half < X < half and -half < Y < half):
                    continue
                if i % 2 == 0 and j % 2 != 0:
                    val = math.cos(X) * math.sin(Y)
                    kind = "max" if val > 0 else "min"
                elif i % 2 != 0 and j % 2 == 0:
                    kind = "saddle"
                else:
                    continue
                gx = (X / L + 0.5) * (self.nx - 1)
                gy = (Y / L + 0.5) * (self.ny - 1)
                out.append((gx, gy, kind))
        return out


@dataclass
class MovingExtremum:
    """f = sum_a sign_a (x_a - c_a(t))^2, c(t) = c0 + v t on integer grid coordinates
    (x_c(t) = x0 + d t).  signs all +1 = moving minimum."""
    n: tuple            # spatial extents (nx, ny[, nz])
    nt: int
    c0: tuple
    v: tuple
    signs: tuple = dc_field(default=None)
    scale_log2: int = 8

    def __post_init__(self):
        if self.signs is None:
            self.signs = (1,) * len(self.n)

    def center(self, t: float):
        return tuple(c + vv * t for c, vv in zip(self.c0, self.v))

    def plane(self, t_global: int, device="cpu") -> torch.Tensor:
        c = self.center(t_global)
        axes = [torch.arange(N, dtype=torch.float64, device=device) for N in self.n]
        if len(self.n) == 2:
            Y, X = torch.meshgrid(axes[1], axes[0], indexing="ij")
            grids = (X, Y)
        else:
            Z, Y, X = torch.meshgrid(axes[2], axes[1], axes[0], indexing="ij")
            grids = (X, Y, Z)
        f = torch.zeros_like(grids[0])
        for g, cc, sg in zip(grids, c, self.signs):
            f = f + sg * (g - cc) ** 2
        return f

    def generate(self, t0: int = 0, nt: int | None = None, device="cpu", dtype=torch.float32):
        nt = self.nt - t0 if nt is None else nt
        shape = (nt,) + tuple(reversed(self.n))
        out = torch.empty(shape, dtype=dtype, device=device)
        for k in range(nt):
            out[k] = self.plane(t0 + k, device).to(dtype)
        return out


@dataclass
class DoubleGyre:
    """2D time-varying vector field [t][y][x][2] (u, v interleaved) of the double gyre (PAPER.md:509-511:
    domain [0,2] x [0,1], timesteps 0.1 apart): u = -pi A sin(pi f) cos(pi y),
    v = pi A cos(pi f) sin(pi y) df/dx, f = a(t) x^2 + b(t) x, a = eps sin(w t), b = 1 - 2 eps sin(w t);
    the common parameters A = 0.1, eps = 0.25, w = 2 pi / 10 (our choice; the paper gives none)."""
    nx: int
    ny: int
    nt: int
    dt: float = 0.1
    A: float = 0.1
    eps: float = 0.25
    omega: float = 2.0 * math.pi / 10.0
    scale_log2: int = 26

    def plane(self, t_global: int, device="cpu") -> torch.Tensor:
        t = t_global * self.dt
        xs = torch.arange(self.nx, dtype=torch.float64, device=device) * (2.0 / (self.nx - 1))
        ys = torch.arange(self.ny, dtype=torch.float64, device=device) * (1.0 / (self.ny - 1))
        Y, X = torch.meshgrid(ys, xs, indexing="ij")
        a = self.eps * math.sin(self.omega * t)
        b = 1.0 - 2.0 * a
        f = a * X * X + b * X
        dfdx = 2.0 * a * X + b
        u = -math.pi * self.A * torch.sin(math.pi * f) * torch.cos(math.pi * Y)
        v = math.pi * self.A * torch.cos(math.pi * f) * torch.sin(math.pi * Y) * dfdx
        return torch.stack([u, v], dim=-1)

    def generate(self, t0: int = 0, nt: int | None = None, device="cpu", dtype=torch.float32):
        nt = self.nt - t0 if nt is None else nt
        out = torch.empty((nt, self.ny, self.nx, 2), dtype=dtype, device=device)
        for k in range(nt):
            out[k] = self.plane(t0 + k, device).to(dtype)
        return out


@dataclass
class MovingLinear:
    """2D vector field v(x, t) = A (x - c(t)), c(t) = c0 + w t, on integer grid coordinates: the PL
    field is exactly linear, so its one zero per timestep is c(t) and its type is A's (source, sink,
    saddle, spiral, centre).  Dyadic c and integer A with scale 2^8 keep every value exact in fp32."""
    n: tuple
    nt: int
    A: tuple            # ((a, b), (c, d))
    c0: tuple
    w: tuple
    scale_log2: int = 8

    def center(self, t: float):
        return tuple(c + vv * t for c, vv in zip(self.c0, self.w))

    def plane(self, t_global: int, device="cpu") -> torch.Tensor:
        cx, cy = self.center(t_global)
        xs = torch.arange(self.n[0], dtype=torch.float64, device=device) - cx
        ys = torch.arange(self.n[1], dtype=torch.float64, device=device) - cy
        Y, X = torch.meshgrid(ys, xs, indexing="ij")
        (a, b), (c, d) = self.A
        return torch.stack([a * X + b * Y, c * X + d * Y], dim=-1)

    def generate(self, t0: int = 0, nt: int | None = None, device="cpu", dtype=torch.float32):
        nt = self.nt - t0 if nt is None else nt
        out = torch.empty((nt, self.n[1], self.n[0], 2), dtype=dtype, device=device)
        for k in range(nt):
            out[k] = self.plane(t0 + k, device).to(dtype)
        return out


@dataclass
class MovingLinear3:
    """3D vector field v(x, t) = A (x - c(t)), [t][z][y][x][3]; as MovingLinear, one zero per timestep
    at c(t), typed by the 3x3 integer matrix A."""
    n: tuple
    nt: int
    A: tuple
    c0: tuple
    w: tuple
    scale_log2: int = 8

    def center(self, t: float):
        return tuple(c + vv * t for c, vv in zip(self.c0, self.w))

    def plane(self, t_global: int, device="cpu") -> torch.Tensor:
        c = self.center(t_global)
        axes = [torch.arange(N, dtype=torch.float64, device=device) - cc for N, cc in zip(self.n, c)]
        Z, Y, X = torch.meshgrid(axes[2], axes[1], axes[0], indexing="ij")
        comps = [self.A[j][0] * X + self.A[j][1] * Y + self.A[j][2] * Z for j in range(3)]
        return torch.stack(comps, dim=-1)

    def generate(self, t0: int = 0, nt: int | None = None, device="cpu", dtype=torch.float32):
        nt = self.nt - t0 if nt is None else nt
        out = torch.empty((nt, self.n[2], self.n[1], self.n[0], 3), dtype=dtype, device=device)
        for k in range(nt):
            out[k] = self.plane(t0 + k, device).to(dtype)
        return out


@dataclass
class ABCFlow:
    """Time-periodic 3D ABC-like flow on [0, 2 pi)^3 grid coordinates (our 3D vector workload; the paper
    shows no 3D vector field): u = A sin z + C cos y, v = B sin x + A cos z, w = C sin y + B cos x, with
    A = sqrt(3) + 0.5 sin(w t), B = sqrt(2), C = 1; stagnation points are isolated and move in time."""
    nx: int
    ny: int
    nz: int
    nt: int
    dt: float = 0.1
    scale_log2: int = 26

    def plane(self, t_global: int, device="cpu") -> torch.Tensor:
        t = t_global * self.dt
        A, B, C = math.sqrt(3.0) + 0.5 * math.sin(2.0 * math.pi * t / 10.0), math.sqrt(2.0), 1.0
        ax = [torch.arange(n, dtype=torch.float64, device=device) * (2.0 * math.pi / n) for n in (self.nx, self.ny, self.nz)]
        Z, Y, X = torch.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
        u = A * torch.sin(Z) + C * torch.cos(Y)
        v = B * torch.sin(X) + A * torch.cos(Z)
        w = C * torch.sin(Y) + B * torch.cos(X)
        return torch.stack([u, v, w], dim=-1)

    def generate(self, t0: int = 0, nt: int | None = None, device="cpu", dtype=torch.float32):
        nt = self.nt - t0 if nt is None else nt
        out = torch.empty((nt, self.nz, self.ny, self.nx, 3), dtype=dtype, device=device)
        for k in range(nt):
            out[k] = self.plane(t0 + k, device).to(dtype)
        return out


def random_degenerate(shape, values=(-1.0, 0.0, 1.0), seed=0, dtype=torch.float32):
    """Massively degenerate field: every vertex value drawn from a tiny set (ties everywhere)."""
    g = torch.Generator().manual_seed(seed)
    idx = torch.randint(0, len(values), shape, generator=g)
    return torch.tensor(values, dtype=torch.float64)[idx].to(dtype)


# --------------------------------------------------------------------------------------------
# Config registry (BASELINE.json configs).
# --------------------------------------------------------------------------------------------
@dataclass
class Config:
    name: str
    kind: str          # woven2d | moving3d | woven3d | gyre2d / abc3d (vector fields)
    shape: tuple       # (nx, ny, [nz,] nt)
    scale_log2: int
    desc: str

    def make(self, nt: int | None = None):
        if self.kind == "woven2d":
            nx, ny, T = self.shape
            return Woven(nx, ny, nt or T, L=15.0 if self.name == "C1" else None, scale_log2=self.scale_log2)
        if self.kind == "woven3d":
            nx, ny, nz, T = self.shape
            return Woven(nx, ny, nt or T, nz=nz, scale_log2=self.scale_log2)
        if self.kind == "abc3d":
            nx, ny, nz, T = self.shape
            return ABCFlow(nx, ny, nz, nt or T, scale_log2=self.scale_log2)
        if self.kind == "gyre2d":
            nx, ny, T = self.shape
            return DoubleGyre(nx, ny, nt or T, scale_log2=self.scale_log2)
        if self.kind == "moving3d":
            nx, ny, nz, T = self.shape
            return MovingExtremum((nx, ny, nz), nt or T, c0=(60.0, 62.0, 64.0), v=(0.25, 0.125, -0.0625),
                                  scale_log2=self.scale_log2)
        raise ValueError(self.kind)


CONFIGS = {
    "C1": Config("C1", "woven2d", (32, 32, 8), 26, "2D woven 32x32x8, L=15 (parity fixture)"),
    "C2": Config("C2", "woven2d", (1024, 1024, 256), 26, "2D woven 1024x1024x256, 1 B200"),
    "C3": Config("C3", "moving3d", (128, 128, 128, 32), 8, "3D moving extremum 128^3x32"),
    "C4": Config("C4", "woven2d", (4096, 4096, 512), 26, "2D woven 4096^2x512, time-slab strong scaling"),
    "C5": Config("C5", "woven3d", (256, 256, 256, 64), 26, "3D woven 256^3x64 per GPU, weak scaling"),
    # SURVEY.md 8(f) NEXT row 2 (vector-field input); not a BASELINE.json config
    "V2": Config("V2", "gyre2d", (2048, 1024, 256), 26, "2D double-gyre vector field 2048x1024x256 (vector path)"),
    "V5": Config("V5", "abc3d", (256, 256, 256, 64), 26, "3D ABC-flow vector field 256^3x64 (3D vector path)"),
}

