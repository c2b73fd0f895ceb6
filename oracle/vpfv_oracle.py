"""numpy restatement of the reference VP-FV stage path -- TEST INFRASTRUCTURE ONLY.

Every function cites the reference file:line (under /root/reference/pkg/src/vpfv)
it restates.  Nothing here is imported by the product package.

Two right-hand-side evaluations are restated because the reference has two:

* ``fused_stage`` -- the numba kernels ``stage_{1d1v,1d2v,2d2v}``
  (``_kernels.py:92-317``), evaluated here with numpy in *exactly* the
  kernels' per-cell operation order.  numba compiles them without FMA and with
  true division, and numpy's elementwise ufuncs round each
  operation once as well, so this restatement is bitwise equal to the numba
  kernels (pinned by ``tests/test_oracle.py`` against reference fixtures).
* ``vlasov_rhs`` -- the numpy production operator (``fvm.py:144-263``) that
  the reference drivers call (``runner.py:186``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

NGHOST = 3  # grid.py:17

# fvm.py:36-37 -- five-point upwind face weights
W_UP = np.array([2.0, -13.0, 47.0, 27.0, -3.0]) / 60.0
W_DN = np.array([-3.0, 27.0, 47.0, -13.0, 2.0]) / 60.0

DEFAULT_SIGMA = 1.73  # timestepping.py:33


# ---------------------------------------------------------------------------
# geometry (grid.py:20-102, 105-150)


@dataclass(frozen=True)
class Grid:
    d: int
    v: int
    N: tuple
    lo: tuple
    hi: tuple
    periodic: tuple = None
    spacing: tuple = None

    def __post_init__(self):
        if self.periodic is None:
            object.__setattr__(self, "periodic", tuple(k < self.d for k in range(self.ndim)))

    @property
    def ndim(self):
        return self.d + self.v

    @property
    def h(self):  # grid.py:51-55
        if self.spacing is not None:
            return tuple(self.spacing)
        return tuple((self.hi[k] - self.lo[k]) / self.N[k] for k in range(self.ndim))

    @property
    def padded_shape(self):
        return tuple(n + 2 * NGHOST for n in self.N)

    def centers(self, dim):  # grid.py:81-84
        return self.lo[dim] + (np.arange(self.N[dim]) + 0.5) * self.h[dim]

    def inner(self):
        return tuple(slice(NGHOST, NGHOST + n) for n in self.N)

    @property
    def velocity_dims(self):
        return tuple(range(self.d, self.ndim))


def grid_from(g):
    """Oracle grid from any object exposing the reference grid attributes."""
    return Grid(g.d, g.v, tuple(g.N), tuple(g.lo), tuple(g.hi), tuple(g.periodic),
                None if getattr(g, "spacing", None) is None else tuple(g.spacing))


@dataclass(frozen=True)
class Species:  # fvm.py:40-59
    name: str = "e"
    q: float = -1.0
    m: float = 1.0
    kappa2: float = 1.0
    kappa_c: float = 0.0
    Bz: float = 0.0
    G: tuple = (0.0,)

    @property
    def qm(self):
        return self.q / self.m


def species_from(s):
    return Species(s.name, s.q, s.m, s.kappa2, s.kappa_c, s.Bz, tuple(s.G))


def _g2(s):  # fvm.py:72-74
    return (tuple(s.G) + (0.0, 0.0))[:2]


# ---------------------------------------------------------------------------
# ghosts (grid.py:215-277)


def capture_frozen(data, g):
    """Velocity-boundary slabs pinned at t=0 (grid.py:227-241)."""
    slabs = {}
    for k in range(g.ndim):
        if g.periodic[k]:
            continue
        n = g.N[k]
        lo = [slice(None)] * g.ndim
        hi = [slice(None)] * g.ndim
        lo[k] = slice(0, NGHOST)
        hi[k] = slice(n + NGHOST, n + 2 * NGHOST)
        slabs[(k, 0)] = data[tuple(lo)].copy()
        slabs[(k, 1)] = data[tuple(hi)].copy()
    return slabs


def fill_ghosts(data, g, frozen=None):
    """Frozen slabs first, then whole-column periodic wraps (grid.py:244-277)."""
    if not all(g.periodic):
        if frozen is None:
            raise ValueError("non-periodic dimensions present but no frozen ghost snapshot")
        for (k, side), slab in frozen.items():
            n = g.N[k]
            sl = [slice(None)] * g.ndim
            sl[k] = slice(0, NGHOST) if side == 0 else slice(n + NGHOST, n + 2 * NGHOST)
            data[tuple(sl)] = slab
    for k in range(g.ndim):
        if not g.periodic[k]:
            continue
        n = g.N[k]
        a = [slice(None)] * g.ndim
        b = [slice(None)] * g.ndim
        a[k] = slice(0, NGHOST)
        b[k] = slice(n, n + NGHOST)
        data[tuple(a)] = data[tuple(b)]
        a[k] = slice(n + NGHOST, n + 2 * NGHOST)
        b[k] = slice(NGHOST, 2 * NGHOST)
        data[tuple(a)] = data[tuple(b)]
    return data


# ---------------------------------------------------------------------------
# speeds and correction coefficients (fvm.py:77-122, 168-201)


def correction_coeffs(g, s, E):
    """fvm.py:168-201, same expression order."""
    h = g.h
    qm = s.qm
    if g.d == 1:
        hx, hvx = h[0], h[1]
        Ex = np.asarray(E["Ex"])
        dEx = np.roll(Ex, -1) - np.roll(Ex, 1)
        c = {"c1": hvx / (48.0 * hx) + qm * s.kappa2 * dEx / (96.0 * hvx)}
        if g.v == 2:
            hvy = h[2]
            c["c2"] = qm * (s.kappa_c / 48.0) * s.Bz * (hvx / hvy - hvy / hvx)
        return c
    hx, hy, hvx, hvy = h
    Ex = np.asarray(E["Ex"])
    Ey = np.asarray(E["Ey"])
    dEx_x = np.roll(Ex, -1, axis=0) - np.roll(Ex, 1, axis=0)
    dEy_y = np.roll(Ey, -1, axis=1) - np.roll(Ey, 1, axis=1)
    dEx_y = np.roll(Ex, -1, axis=1) - np.roll(Ex, 1, axis=1)
    dEy_x = np.roll(Ey, -1, axis=0) - np.roll(Ey, 1, axis=0)
    return {
        "c1": hvx / (48.0 * hx) + qm * s.kappa2 * dEx_x / (96.0 * hvx),
        "c2": qm * (s.kappa_c / 48.0) * s.Bz * (hvx / hvy - hvy / hvx),
        "c3": -qm * s.kappa2 * dEx_y / (96.0 * hvx),
        "c4": hvy / (48.0 * hy) + qm * s.kappa2 * dEy_y / (96.0 * hvy),
        "c5": -qm * s.kappa2 * dEy_x / (96.0 * hvy),
    }


def advection_speeds(g, s, E):
    """Broadcast per-dimension speeds (fvm.py:77-122)."""
    gx, gy = _g2(s)
    cB = s.qm * s.kappa_c * s.Bz
    if (g.d, g.v) == (1, 1):
        return [g.centers(1)[None, :], (s.qm * s.kappa2 * np.asarray(E["Ex"]) + gx)[:, None]]
    if (g.d, g.v) == (1, 2):
        evx = s.qm * s.kappa2 * np.asarray(E["Ex"]) + gx
        return [
            g.centers(1)[None, :, None],
            evx[:, None, None] + cB * g.centers(2)[None, None, :],
            (-cB * g.centers(1) + gy)[None, :, None],
        ]
    if (g.d, g.v) == (2, 2):
        evx = s.qm * s.kappa2 * np.asarray(E["Ex"]) + gx
        evy = s.qm * s.kappa2 * np.asarray(E["Ey"]) + gy
        return [
            g.centers(2)[None, None, :, None],
            g.centers(3)[None, None, None, :],
            evx[:, :, None, None] + cB * g.centers(3)[None, None, None, :],
            evy[:, :, None, None] - cB * g.centers(2)[None, None, :, None],
        ]
    raise ValueError(f"unsupported dimensionality ({g.d},{g.v})")


def max_speed_per_dim(g, s, E):  # fvm.py:125-127
    return [float(np.max(np.abs(a))) for a in advection_speeds(g, s, E)]


# ---------------------------------------------------------------------------
# the numpy production operator (fvm.py:130-263)


def _view(data, g, off):
    return data[tuple(slice(NGHOST + o, NGHOST + o + n) for o, n in zip(off, g.N))]


def _axis(data, g, dim, o):
    z = [0] * g.ndim
    z[dim] = o
    return _view(data, g, z)


def _flux_difference(data, g, dim, A):  # fvm.py:144-153
    h = g.h[dim]
    hi_p = sum(w * _axis(data, g, dim, o) for w, o in zip(W_UP, range(-2, 3)))
    lo_p = sum(w * _axis(data, g, dim, o) for w, o in zip(W_UP, range(-3, 2)))
    hi_n = sum(w * _axis(data, g, dim, o) for w, o in zip(W_DN, range(-1, 4)))
    lo_n = sum(w * _axis(data, g, dim, o) for w, o in zip(W_DN, range(-2, 3)))
    return np.where(A > 0.0, A * (hi_p - lo_p), A * (hi_n - lo_n)) / h


def _diag(data, g, a, b):  # fvm.py:156-165
    def d2(sa, sb):
        z = [0] * g.ndim
        z[a] = sa
        z[b] = sb
        return _view(data, g, z)

    return d2(1, -1) + d2(-1, 1) - d2(1, 1) - d2(-1, -1)


def transverse_correction(data, g, c):  # fvm.py:204-237
    if (g.d, g.v) == (1, 1):
        return c["c1"][:, None] * _diag(data, g, 0, 1)
    if (g.d, g.v) == (1, 2):
        out = c["c1"][:, None, None] * _diag(data, g, 0, 1)
        out -= c["c2"] * _diag(data, g, 1, 2)
        return out
    e = lambda k: c[k][:, :, None, None]  # noqa: E731
    out = e("c1") * _diag(data, g, 0, 2)
    out += e("c4") * _diag(data, g, 1, 3)
    out -= c["c2"] * _diag(data, g, 2, 3)
    out -= e("c3") * _diag(data, g, 1, 2)
    out -= e("c5") * _diag(data, g, 0, 3)
    return out


def vlasov_rhs(data, g, s, E, corrections=True):  # fvm.py:240-263
    speeds = advection_speeds(g, s, E)
    rhs = np.zeros(g.N)
    for dim in range(g.ndim):
        rhs -= _flux_difference(data, g, dim, speeds[dim])
    if corrections:
        rhs += transverse_correction(data, g, correction_coeffs(g, s, E))
    return rhs


# ---------------------------------------------------------------------------
# the fused numba kernels, restated in their per-cell operation order
# (_kernels.py:66-317)


def _fd(data, g, dim, positive):
    """6-point face difference over 60 (_kernels.py:66-89 and 3d/4d twins)."""
    S = lambda o: _axis(data, g, dim, o)  # noqa: E731
    if positive:
        t = -2.0 * S(-3)
        t = t + 15.0 * S(-2)
        t = t - 60.0 * S(-1)
        t = t + 20.0 * S(0)
        t = t + 30.0 * S(1)
        t = t - 3.0 * S(2)
    else:
        t = 3.0 * S(-2)
        t = t - 30.0 * S(-1)
        t = t - 20.0 * S(0)
        t = t + 60.0 * S(1)
        t = t - 15.0 * S(2)
        t = t + 2.0 * S(3)
    return t / 60.0


def _upwind(data, g, dim, a):
    a = np.broadcast_to(a, g.N)
    return np.where(a > 0.0, a * _fd(data, g, dim, True), a * _fd(data, g, dim, False))


def _diag_k(data, g, a, b):
    """(s[+a,-b] + s[-a,+b]) - s[+a,+b] - s[-a,-b], kernel order."""
    def d2(sa, sb):
        z = [0] * g.ndim
        z[a] = sa
        z[b] = sb
        return _view(data, g, z)

    return ((d2(1, -1) + d2(-1, 1)) - d2(1, 1)) - d2(-1, -1)


def stage_tables(g, s, E):
    """Host-side per-line tables the fused dispatcher builds (_kernels.py:330-365)."""
    gx, gy = _g2(s)
    cB = s.qm * s.kappa_c * s.Bz
    c = correction_coeffs(g, s, E)
    if (g.d, g.v) == (1, 1):
        return dict(ax=g.centers(1), avx=s.qm * s.kappa2 * np.asarray(E["Ex"]) + gx, c1=c["c1"])
    if (g.d, g.v) == (1, 2):
        vyc = np.empty(g.N[2] + 1)
        vyc[:-1] = g.centers(2)
        vyc[-1] = cB
        return dict(vxc=g.centers(1), vyc=vyc,
                    evx=s.qm * s.kappa2 * np.asarray(E["Ex"]) + gx,
                    avy=-cB * g.centers(1) + gy, c1=c["c1"], c2=float(c["c2"]))
    return dict(vxc=g.centers(2), vyc=g.centers(3),
                evx=s.qm * s.kappa2 * np.asarray(E["Ex"]) + gx,
                evy=s.qm * s.kappa2 * np.asarray(E["Ey"]) + gy, cB=cB,
                c1=c["c1"], c2=float(c["c2"]), c3=c["c3"], c4=c["c4"], c5=c["c5"])


def slice_tables(T, x0, nloc):
    """Per-slab view of global line tables (runner.py:398-429: coefficients
    come from the global E and are sliced per box)."""
    out = dict(T)
    for k in ("avx", "evx", "evy", "c1", "c3", "c4", "c5"):
        if k in out and isinstance(out[k], np.ndarray):
            out[k] = out[k][x0:x0 + nloc]
    return out


def fused_rhs(src, g, s, E, T=None):
    """RHS exactly as the fused kernels accumulate it (_kernels.py:97-113,
    167-194, 264-313).  ``T`` optionally supplies precomputed tables."""
    if T is None:
        T = stage_tables(g, s, E)
    h = g.h
    if (g.d, g.v) == (1, 1):
        a_x = T["ax"][None, :]
        a_v = T["avx"][:, None]
        rhs = (-np.broadcast_to(a_x, g.N) * _fd_sel(src, g, 0, a_x)) / h[0]
        rhs = rhs - (np.broadcast_to(a_v, g.N) * _fd_sel(src, g, 1, a_v)) / h[1]
        rhs = rhs + T["c1"][:, None] * _diag_k(src, g, 0, 1)
        return rhs
    if (g.d, g.v) == (1, 2):
        cB = T["vyc"][-1]
        a_x = T["vxc"][None, :, None]
        a_vx = T["evx"][:, None, None] + cB * T["vyc"][:-1][None, None, :]
        a_vy = T["avy"][None, :, None]
        rhs = (-np.broadcast_to(a_x, g.N) * _fd_sel(src, g, 0, a_x)) / h[0]
        rhs = rhs - (np.broadcast_to(a_vx, g.N) * _fd_sel(src, g, 1, a_vx)) / h[1]
        rhs = rhs - (np.broadcast_to(a_vy, g.N) * _fd_sel(src, g, 2, a_vy)) / h[2]
        rhs = rhs + T["c1"][:, None, None] * _diag_k(src, g, 0, 1)
        rhs = rhs - T["c2"] * _diag_k(src, g, 1, 2)
        return rhs
    cB = T["cB"]
    vxc, vyc = T["vxc"], T["vyc"]
    a_x = vxc[None, None, :, None]
    a_y = vyc[None, None, None, :]
    a_vx = T["evx"][:, :, None, None] + cB * vyc[None, None, None, :]
    a_vy = T["evy"][:, :, None, None] - cB * vxc[None, None, :, None]
    rhs = (-np.broadcast_to(a_x, g.N) * _fd_sel(src, g, 0, a_x)) / h[0]
    rhs = rhs - (np.broadcast_to(a_y, g.N) * _fd_sel(src, g, 1, a_y)) / h[1]
    rhs = rhs - (np.broadcast_to(a_vx, g.N) * _fd_sel(src, g, 2, a_vx)) / h[2]
    rhs = rhs - (np.broadcast_to(a_vy, g.N) * _fd_sel(src, g, 3, a_vy)) / h[3]
    e = lambda k: T[k][:, :, None, None]  # noqa: E731
    rhs = rhs + e("c1") * _diag_k(src, g, 0, 2)
    rhs = rhs + e("c4") * _diag_k(src, g, 1, 3)
    rhs = rhs - T["c2"] * _diag_k(src, g, 2, 3)
    rhs = rhs - e("c3") * _diag_k(src, g, 1, 2)
    rhs = rhs - e("c5") * _diag_k(src, g, 0, 3)
    return rhs


def _fd_sel(data, g, dim, a):
    a = np.broadcast_to(a, g.N)
    return np.where(a > 0.0, _fd(data, g, dim, True), _fd(data, g, dim, False))


def first_nonfinite(dest, g):
    """Interior multi-index of the first non-finite value (_kernels.py:33-60,
    368-373), or None."""
    bad = ~np.isfinite(dest[g.inner()])
    if not bad.any():
        return None
    return tuple(int(i) for i in np.unravel_index(np.argmax(bad), g.N))


def fused_stage(dest, A, B, src, ca, cb, cd, cL, g, s, E, check=True, tables=None):
    """``fused_stage`` (_kernels.py:320-373): in-place interior update."""
    if dest is src:
        raise ValueError("dest must not alias src")
    if (g.d, g.v) not in ((1, 1), (1, 2), (2, 2)):
        raise ValueError(f"unsupported dimensionality ({g.d},{g.v})")
    inner = g.inner()
    rhs = fused_rhs(src, g, s, E, tables)
    dest[inner] = ((ca * A[inner] + cb * B[inner]) + cd * dest[inner]) + cL * rhs
    if check:
        mi = first_nonfinite(dest, g)
        if mi is not None:
            raise FloatingPointError(f"non-finite stage output at interior index {mi}")


# ---------------------------------------------------------------------------
# moments, charge density, Poisson (fields.py:28-213)


def fold_axis(x, axis):  # fields.py:28-39
    x = np.moveaxis(x, axis, -1)
    n = x.shape[-1]
    while n > 1:
        m = n // 2
        s = x[..., 0:2 * m:2] + x[..., 1:2 * m:2]
        if n % 2:
            s = np.concatenate([s, x[..., 2 * m:]], axis=-1)
        x = s
        n = x.shape[-1]
    return np.moveaxis(x, -1, axis)


def fold_tree_sum(x, axes):  # fields.py:42-47
    out = np.array(x, dtype=np.float64, copy=True)
    for ax in sorted(axes, reverse=True):
        out = fold_axis(out, ax)
    return np.squeeze(out, axis=tuple(sorted(axes)))


def velocity_volume(g):
    vol = 1.0
    for k in g.velocity_dims:
        vol *= g.h[k]
    return vol


def zeroth_moment(data, g, schedule="velocity-major"):  # fields.py:86-111
    interior = data[g.inner()]
    vol = velocity_volume(g)
    if schedule == "velocity-major":
        n = fold_tree_sum(interior, g.velocity_dims)
    elif schedule == "position-major":  # _seq_moment_{2,3,4}d (fields.py:50-83): s += f in C order
        flat = interior.reshape(tuple(g.N[:g.d]) + (-1,))
        n = np.add.accumulate(flat, axis=-1)[..., -1]  # strictly sequential, left to right
    elif schedule == "free":
        n = interior.sum(axis=g.velocity_dims)
    else:
        raise ValueError(f"unknown schedule {schedule!r}")
    return n * vol


def charge_density(densities, species):  # fields.py:164-169
    rho = None
    for n_s, sp in zip(densities, species):
        rho = sp.q * n_s if rho is None else rho + sp.q * n_s
    return rho - np.mean(rho)


def poisson_solve(rho, g):  # fields.py:172-213
    rho = np.asarray(rho)
    d = g.d
    if rho.ndim != d:
        raise ValueError("charge density must live on the physical grid")
    scale = np.max(np.abs(rho)) if rho.size else 0.0
    if abs(np.mean(rho)) > 1e-10 * max(scale, 1.0):
        raise ValueError("poisson_solve requires zero-mean charge density")
    ks = [2.0 * np.pi * np.fft.fftfreq(g.N[i], d=g.h[i]) for i in range(d)]
    if d == 1:
        k = ks[0]
        rhohat = np.fft.fft(rho)
        k2 = k ** 2
        phihat = np.zeros_like(rhohat)
        phihat[1:] = rhohat[1:] / k2[1:]
        kd = k.copy()
        if g.N[0] % 2 == 0:
            kd[g.N[0] // 2] = 0.0
        Ehat = -1j * kd * phihat
        return np.fft.ifft(phihat).real, {"Ex": np.fft.ifft(Ehat).real}
    kx = ks[0][:, None]
    ky = ks[1][None, :]
    rhohat = np.fft.fftn(rho)
    k2 = kx ** 2 + ky ** 2
    phihat = np.where(k2 > 0.0, rhohat / np.where(k2 > 0.0, k2, 1.0), 0.0)
    kxd, kyd = kx.copy(), ky.copy()
    if g.N[0] % 2 == 0:
        kxd[g.N[0] // 2, 0] = 0.0
    if g.N[1] % 2 == 0:
        kyd[0, g.N[1] // 2] = 0.0
    Ex = np.fft.ifftn(-1j * kxd * phihat).real
    Ey = np.fft.ifftn(-1j * kyd * phihat).real
    return np.fft.ifftn(phihat).real, {"Ex": Ex, "Ey": Ey}


def field_solve(datas, grids, species, schedule="velocity-major"):
    """FieldState.solve (fields.py:226-239): densities -> rho -> E."""
    dens = [zeroth_moment(a, g, schedule) for a, g in zip(datas, grids)]
    rho = charge_density(dens, species)
    _, E = poisson_solve(rho, grids[0])
    return dens, rho, E


# ---------------------------------------------------------------------------
# time stepping (timestepping.py:39-117, runner.py:98-103)


@dataclass
class StepContext:  # timestepping.py:39-52
    f0: object
    f1: object
    fout: object
    t: float = 0.0
    step: int = 0

    def rotate(self):
        self.f0, self.fout = self.fout, self.f0
        self.step += 1


RK_STAGES = (  # timestepping.py:80-83: (dest, A, B, src, ca, cb, cd, cL/dt)
    ("f1", "f0", "f0", "f0", 1.0, 0.0, 0.0, 1.0 / 3.0),
    ("fout", "f0", "f1", "f1", 2.0, -1.0, 0.0, 1.0),
    ("f1", "fout", "fout", "fout", -1.0, 0.0, 2.0, 1.0),
    ("fout", "f0", "f1", "f1", -0.125, 0.375, 0.75, 0.125),
)


def rk4_38_low_storage_step(ctx, dt, stage):  # timestepping.py:69-84
    f0, f1, fout = ctx.f0, ctx.f1, ctx.fout
    t = ctx.t
    stage(f1, f0, f0, f0, 1.0, 0.0, 0.0, dt / 3.0, t)
    stage(fout, f0, f1, f1, 2.0, -1.0, 0.0, dt, t + dt / 3.0)
    stage(f1, fout, fout, fout, -1.0, 0.0, 2.0, dt, t + 2.0 * dt / 3.0)
    stage(fout, f0, f1, f1, -0.125, 0.375, 0.75, dt / 8.0, t + dt)
    ctx.t = t + dt


def rk4_butcher_step(u0, dt, L, t=0.0):  # timestepping.py:55-66
    u0 = np.asarray(u0)
    k1 = L(u0, t)
    k2 = L(u0 + (dt / 3.0) * k1, t + dt / 3.0)
    k3 = L(u0 + dt * (-k1 / 3.0 + k2), t + 2.0 * dt / 3.0)
    k4 = L(u0 + dt * (k1 - k2 + k3), t + dt)
    return u0 + (dt / 8.0) * (k1 + 3.0 * k2 + 3.0 * k3 + k4)


def max_stable_dt(speeds, h, sigma=DEFAULT_SIGMA, safety=1.0):  # timestepping.py:101-117
    best = math.inf
    for per_dim in speeds:
        if len(per_dim) != len(h):
            raise ValueError("speed/width dimension mismatch")
        norm1 = sum(abs(a) / hd for a, hd in zip(per_dim, h))
        if norm1 > 0.0:
            best = min(best, sigma / norm1)
    return best * safety if best != math.inf else math.inf


def stable_dt(grids, species, E, sigma=DEFAULT_SIGMA):  # runner.py:98-103
    return min(max_stable_dt([max_speed_per_dim(g, s, E)], g.h, sigma=sigma)
               for g, s in zip(grids, species))


class OracleDiverged(RuntimeError):
    pass


class OracleSimulation:
    """The single-rank driver pipeline (runner.py:126-227).

    ``rhs="numpy"`` is the production operator the reference drivers call
    (runner.py:186); ``rhs="fused"`` routes every stage through the fused
    kernels' arithmetic (the survey's numba-driven variant).
    """

    def __init__(self, grids, species, datas, dt=None, cfl_fraction=0.9,
                 corrections=True, schedule="velocity-major", sigma=DEFAULT_SIGMA,
                 rhs="numpy"):
        self.grids = [grid_from(g) for g in grids]
        self.species = [species_from(s) for s in species]
        self.frozen = [capture_frozen(np.asarray(a), g) for a, g in zip(datas, self.grids)]
        f0 = [np.array(a, dtype=np.float64, copy=True) for a in datas]
        self.ctx = StepContext(f0=f0, f1=[np.zeros_like(a) for a in f0],
                               fout=[np.zeros_like(a) for a in f0])
        self.fixed_dt = dt
        self.cfl_fraction = cfl_fraction
        self.corrections = corrections
        self.schedule = schedule
        self.sigma = sigma
        self.rhs = rhs
        self.last_E = None

    def _solve(self, arrays):
        for a, g, fr in zip(arrays, self.grids, self.frozen):
            fill_ghosts(a, g, fr)
        return field_solve(arrays, self.grids, self.species, self.schedule)

    def _stage(self, dest, A, B, src, ca, cb, cd, cL, t):  # runner.py:183-191
        _, _, E = self._solve(src)
        self.last_E = E
        for s, (g, sp) in enumerate(zip(self.grids, self.species)):
            inner = g.inner()
            if self.rhs == "numpy":
                rhs = vlasov_rhs(src[s], g, sp, E, self.corrections)
                dest[s][inner] = ca * A[s][inner] + cb * B[s][inner] + cd * dest[s][inner] + cL * rhs
            else:
                fused_stage(dest[s], A[s], B[s], src[s], ca, cb, cd, cL, g, sp, E, check=False)

    def max_dt(self):
        _, _, E = self._solve(self.ctx.f0)
        return stable_dt(self.grids, self.species, E, self.sigma)

    def current_dt(self):
        if self.fixed_dt is not None:
            return self.fixed_dt
        return self.max_dt() * self.cfl_fraction

    def advance(self, dt):  # runner.py:219-227
        rk4_38_low_storage_step(self.ctx, dt, self._stage)
        self.ctx.rotate()
        for s, a in enumerate(self.ctx.f0):
            if not math.isfinite(float(np.sum(a[self.grids[s].inner()]))):
                self.ctx.f0, self.ctx.fout = self.ctx.fout, self.ctx.f0
                self.ctx.t -= dt
                self.ctx.step -= 1
                raise OracleDiverged(f"species {s} non-finite")

    def interiors(self):
        return [a[g.inner()].copy() for a, g in zip(self.ctx.f0, self.grids)]

    def field_amplitude(self):
        """sqrt(integral E.E dx) of the current state (diagnostics.py:74-82)."""
        _, _, E = self._solve(self.ctx.f0)
        g = self.grids[0]
        vol = 1.0
        for k in range(g.d):
            vol *= g.h[k]
        return math.sqrt(sum(float(np.sum(np.square(c))) for c in E.values()) * vol)


# ---------------------------------------------------------------------------
# deterministic cross-partition combine (partition.py:778-809)


def combine_partials(partials):
    items = list(partials)
    while len(items) > 1:
        nxt = [items[2 * i] + items[2 * i + 1] for i in range(len(items) // 2)]
        if len(items) % 2:
            nxt.append(items[-1])
        items = nxt
    return items[0]


# ---------------------------------------------------------------------------
# growth-rate fit on field-amplitude peaks (what SURVEY.md section 6 used)


def fit_peak_rate(ts, amps, t_min=0.0, t_max=np.inf):
    """Least-squares slope of log|E| through the local maxima of |E|(t)."""
    ts = np.asarray(ts)
    a = np.asarray(amps)
    idx = [i for i in range(1, len(a) - 1) if a[i] >= a[i - 1] and a[i] > a[i + 1]
           and t_min <= ts[i] <= t_max]
    if len(idx) < 2:
        raise ValueError("not enough peaks to fit")
    return float(np.polyfit(ts[idx], np.log(a[idx]), 1)[0])


def fit_window_rate(ts, amps, t_min, t_max):
    """Plain LS slope of log|E| over a window (growth-phase fits)."""
    ts = np.asarray(ts)
    a = np.asarray(amps)
    m = (ts >= t_min) & (ts <= t_max)
    return float(np.polyfit(ts[m], np.log(a[m]), 1)[0])
